"""Markdown table of an ncu `--metrics ... --csv --log-file F` launch list (every launch, or the
second half with --last-half: the second of two identical calls).  Usage:
python scripts/launch_summary.py F.csv [--last-half]"""
import collections
import csv
import io
import sys

T = {"ns": 1e-6, "nsecond": 1e-6, "us": 1e-3, "usecond": 1e-3, "ms": 1.0, "msecond": 1.0}
B = {"byte": 1e-6, "Kbyte": 1e-3, "Mbyte": 1.0, "Gbyte": 1e3}
lines = [l for l in open(sys.argv[1]) if l.startswith('"')]
r = list(csv.reader(io.StringIO("".join(lines))))
h = r[0]
L = collections.OrderedDict()
for row in r[1:]:
    d = dict(zip(h, row))
    L.setdefault((int(d["ID"]), d["Kernel Name"].split("(")[0].split("::")[-1]), {})[d["Metric Name"]] = (
        float(d["Metric Value"].replace(",", "")), d["Metric Unit"])
items = list(L.items())
if "--last-half" in sys.argv:
    items = items[len(items) // 2:]


def get(v, m, tab):
    x = v.get(m)
    return None if x is None else x[0] * tab.get(x[1], 1.0)


tot = sum(get(v, "gpu__time_duration.sum", T) for _, v in items)
print("| kernel | ms | DRAM read MB | DRAM write MB | warp-instr (M) | issue active % | share |")
print("|---|---|---|---|---|---|---|")
for (i, name), v in items:
    t = get(v, "gpu__time_duration.sum", T)
    rd, wr = get(v, "dram__bytes_read.sum", B), get(v, "dram__bytes_write.sum", B)
    ins = v.get("sm__inst_executed.sum", (float("nan"),))[0] / 1e6
    ia = v.get("smsp__issue_active.avg.pct_of_peak_sustained_active", (float("nan"),))[0]
    print(f"| `{name}` | {t:.3f} | {rd or 0:.1f} | {wr or 0:.1f} | {ins:.1f} | {ia:.1f} | {t / tot * 100:.1f}% |")
print(f"\n{len(items)} launches, {tot:.3f} ms of kernel time (cold-cache, serialised under ncu).")
