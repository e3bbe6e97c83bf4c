"""Rebuild the committed round-2 profile files from a capture (scripts/capture_r02.sh outputs in
gpurun_out/): the bench line, the launch list with the live breakdown, the ncu --set full summaries
and raw pages (headline kernels, the paper's Kelley passes, the fused LMS pass) and the per-launch
DRAM traffic the bench's roofline quotes.  Usage: python scripts/refresh_profiles.py [gpurun_out]"""
import csv
import io
import json
import os
import shutil
import subprocess
import sys

src = sys.argv[1] if len(sys.argv) > 1 else "gpurun_out"
P = "profiles"


def run(*cmd):
    return subprocess.run(list(cmd), capture_output=True, text=True).stdout


def summary(rep, title, md, raw):
    with open(os.path.join(P, md), "w") as f:
        f.write(run(sys.executable, "scripts/ncu_summary.py", os.path.join(src, rep), title))
    with open(os.path.join(P, raw), "w") as f:
        f.write(run("ncu", "-i", os.path.join(src, rep), "--page", "raw", "--csv"))


shutil.copy(os.path.join(src, "r02_bench.json"), os.path.join(P, "r02_bench_single_gpu.json"))
summary("r02_full.ncu-rep", "Round 2 — headline kernels (median of 2^30 float32)", "r02_ncu_headline.md",
        "r02_ncu_full_raw.csv")
summary("r02_kelley.ncu-rep", "Round 2 — the paper's method: Kelley passes from [x_(1), x_(n)] at 2^30 float32 "
        "(init_cut=0 pass_cuts=0 objective=1)", "r02_ncu_kelley.md", "r02_ncu_kelley_raw.csv")
summary("r02_lmsf.ncu-rep", "Round 2 — fused LMS pass (configs[4])", "r02_ncu_lms_fused.md", "r02_ncu_lmsf_raw.csv")

# per-launch DRAM bytes of the headline kernels (the bench's roofline.traffic)
rows = list(csv.reader(open(os.path.join(P, "r02_ncu_full_raw.csv"))))
hdr, units = rows[0], rows[1]
scale = {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9}
tj = {}
for r in rows[2:]:
    d = dict(zip(hdr, r))
    name = d["Kernel Name"].split("(")[0].split("<")[0].replace("void ", "").split("::")[-1]
    b = 0.0
    for k in ("dram__bytes_read.sum", "dram__bytes_write.sum"):
        b += float(d[k].replace(",", "")) * scale.get(units[hdr.index(k)], 1)
    e = tj.setdefault(name, {"dram_bytes_per_launch": 0.0, "launches": 0,
                             "source": "profiles/r02_ncu_full_raw.csv (ncu --set full, dram__bytes_read.sum + "
                                       "dram__bytes_write.sum)"})
    e["dram_bytes_per_launch"] = (e["dram_bytes_per_launch"] * e["launches"] + b) / (e["launches"] + 1)
    e["launches"] += 1
json.dump(tj, open(os.path.join(P, "ncu_pass_traffic.json"), "w"), indent=1)

# launch list + the live breakdown
b = json.load(open(os.path.join(P, "r02_bench_single_gpu.json")))
km = b["kernel_ms_per_step"]
table = open(os.path.join(src, "r02_launch_table.md")).read().strip()
with open(os.path.join(P, "r02_launch_list.md"), "w") as f:
    f.write(f"""# Round 2 — launch list of one timed bench step

Command (one B200; cold-cache and serialised, so shares — not absolute times — compare with the live bench):

```
ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none --csv \\
    --log-file r02_launches.csv python bench.py --steps 1 --warmup 3 --no-e2e --no-cpu --no-lms --no-side
python scripts/launch_table.py r02_launches.csv --sel 4          # (scripts/capture_r02.sh)
```

The timed step = 4 medians of 2^30 float32 (uniform, normal, Cauchy, dup256). Per selection: the
strided-sample gather (all SMs), the 8-CTA cluster select of the two cuts (R29), the fused init pass
(a1 + R23 cuts + a4 copy of ]t_lo, t_hi[ + the value-bin counts of that copy, R38), then — chained
on the device with programmatic dependent launch, no host round trip — the value-binned exact finish
over the ~1% copy (a5: one read of the copy, a shared-memory select of the target bin). 4 launches
per selection.

{table}

Live bench (`profiles/r02_bench_single_gpu.json`, CUDA events, ms per step of 4 selections):
{b['ms_per_step']:.3f} ms; init {km['init']:.3f}, exact finish {km['select']:.3f}, sample kernels {km['sample']:.3f};
{b['value']:.3g} elements/s; init_seg_kernel at {b['roofline']['achieved']:.0f} GB/s = {b['roofline']['frac']:.2f} of the
measured copy peak; the whole call (all algorithmic bytes / step time) {b['whole_call_roofline']['frac']:.2f}.
Earlier in round 2: 2.932 ms (key-digit cooperative radix select, 0.141 ms); round 1: 3.03 ms.
""")
print("refreshed", sorted(os.listdir(P)))
