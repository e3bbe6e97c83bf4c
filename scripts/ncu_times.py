"""Print kernel name + duration (us) + DRAM bytes from an ncu --csv metrics log (stdin)."""
import csv
import sys

rows = [r for r in csv.reader(l for l in sys.stdin if l.startswith('"'))]
hdr = rows[0]
ix = {k: hdr.index(k) for k in ("ID", "Kernel Name", "Metric Name", "Metric Unit", "Metric Value")}
for r in rows[1:]:
    name = r[ix["Kernel Name"]].split("(")[0].replace("void ", "").replace("cpsel::<unnamed>::", "")
    print(f'{r[ix["ID"]]:>4} {name:40s} {r[ix["Metric Name"]]:28s} {r[ix["Metric Value"]]:>14} {r[ix["Metric Unit"]]}')
