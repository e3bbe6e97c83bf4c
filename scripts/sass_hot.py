"""Top SASS lines of one kernel in an ncu source page (ncu -i R --page source --csv --print-source sass):
instructions executed and stall samples, plus region totals between given address markers.
Usage: python scripts/sass_hot.py sass.csv [N]"""
import csv
import sys

rows = list(csv.reader(open(sys.argv[1])))
hdr = rows[1]
ix = {h: i for i, h in enumerate(hdr)}
data = [r for r in rows[2:] if r and r[0].startswith("0x") and len(r) >= len(hdr) - 1]
N = int(sys.argv[2]) if len(sys.argv) > 2 else 40
tot_ins = sum(int(r[ix["Instructions Executed"]] or 0) for r in data)
tot_smp = sum(int(r[ix["Warp Stall Sampling (All Samples)"]] or 0) for r in data)
print(f"total warp-instructions {tot_ins:.4g}, stall samples {tot_smp}")
stall_cols = [h for h in hdr if h.startswith("stall_")]
for k, r in enumerate(data):
    r.append(k)
top = sorted(data, key=lambda r: -int(r[ix["Warp Stall Sampling (All Samples)"]] or 0))[:N]
for r in sorted(top, key=lambda r: r[-1]):
    st = sorted(((int(r[ix[c]] or 0), c[6:]) for c in stall_cols), reverse=True)[:2]
    print(f"{r[-1]:5d} {int(r[ix['Instructions Executed']] or 0):>11d} {int(r[ix['Warp Stall Sampling (All Samples)']] or 0):>6d} "
          f"{r[ix['Source']].strip()[:60]:60s} {st}")
