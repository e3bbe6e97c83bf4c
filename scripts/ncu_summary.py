"""Summarise an ncu report (raw page) into a markdown table: per launch duration, DRAM bytes,
achieved DRAM bandwidth, issue activity, occupancy, top stall reasons."""
import csv
import io
import subprocess
import sys


def rows(rep):
    out = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
    r = list(csv.reader(io.StringIO(out)))
    hdr = r[0]
    return [dict(zip(hdr, x)) for x in r[2:]]


def f(d, k):
    try:
        return float(d.get(k, "nan").replace(",", ""))
    except ValueError:
        return float("nan")


def main(rep, title):
    print(f"### {title}\n\nsource: `{rep}` (ncu --set full --clock-control none)\n")
    print("| # | kernel | grid | regs | duration us | DRAM read GB | DRAM write GB | DRAM GB/s | issue active % | warps active % | top stalls (per issue) |")
    print("|---|---|---|---|---|---|---|---|---|---|---|")
    for i, d in enumerate(rows(rep)):
        name = d["Kernel Name"].split("(")[0].replace("void ", "").replace("(anonymous namespace)::", "")[:48]
        dur = f(d, "gpu__time_duration.sum")
        unit_ms = dur  # ms in raw page
        rd, wr = f(d, "dram__bytes_read.sum"), f(d, "dram__bytes_write.sum")
        gbps = (rd + wr) / (unit_ms / 1e3) if unit_ms else float("nan")
        st = sorted(((k.replace("smsp__average_warps_issue_stalled_", "").replace("_per_issue_active.ratio", ""), f(d, k))
                     for k in d if k.startswith("smsp__average_warps_issue_stalled_") and k.endswith("_per_issue_active.ratio")),
                    key=lambda x: -x[1])[:3]
        print(f"| {i} | `{name}` | {d.get('launch__grid_size')} | {d.get('launch__registers_per_thread')} | {unit_ms*1e3:.1f} | "
              f"{rd:.3f} | {wr:.3f} | {gbps:.0f} | {f(d, 'sm__inst_issued.avg.pct_of_peak_sustained_active'):.1f} | "
              f"{f(d, 'sm__warps_active.avg.pct_of_peak_sustained_active'):.1f} | "
              + ", ".join(f"{k} {v:.2f}" for k, v in st) + " |")


if __name__ == "__main__":
    main(sys.argv[1], sys.argv[2] if len(sys.argv) > 2 else sys.argv[1])
