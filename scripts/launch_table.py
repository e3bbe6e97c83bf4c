"""Markdown table of a `ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum
--csv --log-file F python bench.py --steps 1 ...` launch list: per kernel launches, time, DRAM bytes,
share of the step, for the launches of the LAST `--sel` selections (the timed step).
Usage: python scripts/launch_table.py F.csv [--sel 4]"""
import collections
import csv
import io
import sys

SCALE = {"nsecond": 1e-9, "usecond": 1e-6, "msecond": 1e-3, "second": 1.0, "ns": 1e-9, "us": 1e-6, "ms": 1e-3,
         "byte": 1.0, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9}

path = sys.argv[1]
nsel = int(sys.argv[sys.argv.index("--sel") + 1]) if "--sel" in sys.argv else 4
lines = [l for l in open(path) if l.startswith('"')]
r = list(csv.reader(io.StringIO("".join(lines))))
h = r[0]
launches = collections.OrderedDict()
for row in r[1:]:
    d = dict(zip(h, row))
    key = (int(d["ID"]), d["Kernel Name"])
    launches.setdefault(key, {})[d["Metric Name"]] = float(d["Metric Value"].replace(",", "")) * SCALE.get(d["Metric Unit"], 1)
items = list(launches.items())
def short(n):
    return n.split("(")[0].replace("void ", "").split("::")[-1]


inits = [i for i, ((_, n), _) in enumerate(items) if short(n).startswith(("init_seg_kernel", "init_kernel"))]
# a selection starts at the sample kernels launched just before its init kernel
first = inits[-nsel]
while first > 0 and short(items[first - 1][0][1]).startswith(("sample", "pool_gather")):
    first -= 1
sel = items[first:]
tot = sum(m["gpu__time_duration.sum"] for _, m in sel)
agg = collections.OrderedDict()
for (_, name), m in sel:
    k = name.split("(")[0].replace("void ", "").replace("cpsel::<unnamed>::", "")
    a = agg.setdefault(k, [0, 0.0, 0.0, 0.0, 1e9])
    a[0] += 1
    a[1] += m["gpu__time_duration.sum"]
    a[2] += m.get("dram__bytes_read.sum", 0.0)
    a[3] += m.get("dram__bytes_write.sum", 0.0)
    a[4] = min(a[4], m["gpu__time_duration.sum"])
print("| kernel | launches | total us | mean us | min us | DRAM read MB | DRAM write MB | share |")
print("|---|---|---|---|---|---|---|---|")
for k, a in sorted(agg.items(), key=lambda kv: -kv[1][1]):
    print(f"| `{k}` | {a[0]} | {a[1] * 1e6:.1f} | {a[1] / a[0] * 1e6:.1f} | {a[4] * 1e6:.1f} | {a[2] / 1e6:.1f} | "
          f"{a[3] / 1e6:.1f} | {a[1] / tot * 100:.1f}% |")
print(f"\n{len(sel)} launches, {tot * 1e3:.3f} ms of kernel time over the last {nsel} selections.")
