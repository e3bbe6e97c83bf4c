# A/B over libcpsel variants: ab.sh script.py variant...   (each variant = paper_1104_2732_b200/libcpsel_<v>.so, "base" = libcpsel.so)
S=$1; shift
cp paper_1104_2732_b200/libcpsel.so /tmp/libcpsel_base.so
for v in "$@"; do
  if [ "$v" = base ]; then cp /tmp/libcpsel_base.so paper_1104_2732_b200/libcpsel.so; else cp paper_1104_2732_b200/libcpsel_$v.so paper_1104_2732_b200/libcpsel.so; fi
  python $S $v
done
cp /tmp/libcpsel_base.so paper_1104_2732_b200/libcpsel.so
