"""Group the SASS lines of the first kernel in an ncu source CSV (--page source --print-source sass)
into runs of equal execution count: instructions executed and stall samples per run.
Usage: python scripts/sass_regions.py sass.csv [min_warp_instructions]"""
import csv
import sys

rows = list(csv.reader(open(sys.argv[1])))
hdr = rows[1]
ix = {h: i for i, h in enumerate(hdr)}
data = []
for r in rows[2:]:
    if r and r[0].startswith("0x"):
        data.append(r)
    elif data and r and r[0] == "Kernel Name":
        break
thr = float(sys.argv[2]) if len(sys.argv) > 2 else 1e6
stall_cols = [h for h in hdr if h.startswith("stall_") and "Not Issued" not in h]
tot = sum(int(r[ix["Instructions Executed"]] or 0) for r in data)
tots = sum(int(r[ix["Warp Stall Sampling (All Samples)"]] or 0) for r in data)
print(f"total warp-instructions {tot/1e6:.1f}M, stall samples {tots}")
cur = None
out = []
for k, r in enumerate(data):
    n = int(r[ix["Instructions Executed"]] or 0)
    s = int(r[ix["Warp Stall Sampling (All Samples)"]] or 0)
    st = {c: int(r[ix[c]] or 0) for c in stall_cols}
    if cur and cur["n"] == n:
        cur["len"] += 1; cur["s"] += s; cur["sum"] += n
        for c in st: cur["st"][c] += st[c]
    else:
        if cur: out.append(cur)
        cur = {"k": k, "n": n, "len": 1, "s": s, "sum": n, "src": r[1].strip()[:50], "st": st}
out.append(cur)
for c in out:
    if c["sum"] >= thr or c["s"] > tots * 0.01:
        top = sorted(((v, k[6:]) for k, v in c["st"].items()), reverse=True)[:2]
        print(f"{c['k']:5d} x{c['len']:4d} exec {c['n']:>10d} = {c['sum']/1e6:7.1f}M  samples {c['s']:6d} ({100*c['s']/tots:4.1f}%)  {c['src']:50s} {top}")
