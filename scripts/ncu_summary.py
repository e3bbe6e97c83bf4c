"""Summarise an ncu report (raw page) into a markdown table: per launch duration, DRAM bytes,
achieved DRAM bandwidth, issue activity, occupancy, top stall reasons.
Usage: python scripts/ncu_summary.py REPORT.ncu-rep "title" """
import csv
import io
import subprocess
import sys

SCALE = {"ns": 1e-9, "us": 1e-6, "usecond": 1e-6, "nsecond": 1e-9, "ms": 1e-3, "msecond": 1e-3, "s": 1.0,
         "byte": 1.0, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9, "Tbyte": 1e12, "KB": 1e3, "MB": 1e6, "GB": 1e9}


def rows(rep):
    out = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
    r = list(csv.reader(io.StringIO(out)))
    hdr, units = r[0], r[1]
    return [(dict(zip(hdr, x)), dict(zip(hdr, units))) for x in r[2:]]


def val(d, u, k):
    try:
        v = float(d.get(k, "nan").replace(",", ""))
    except ValueError:
        return float("nan")
    return v * SCALE.get(u.get(k, ""), 1.0)


def main(rep, title):
    print(f"### {title}\n\nsource: `{rep}` (ncu --set full --clock-control none)\n")
    print("| # | kernel | grid | regs | duration us | DRAM read MB | DRAM write MB | DRAM GB/s | issue active % | "
          "warps active % | top stalls (per issue) |")
    print("|---|---|---|---|---|---|---|---|---|---|---|")
    for i, (d, u) in enumerate(rows(rep)):
        name = d["Kernel Name"].split("(")[0].replace("void ", "").replace("cpsel::<unnamed>::", "")[:44]
        dur = val(d, u, "gpu__time_duration.sum")
        rd, wr = val(d, u, "dram__bytes_read.sum"), val(d, u, "dram__bytes_write.sum")
        gbps = (rd + wr) / dur / 1e9 if dur else float("nan")
        st = sorted(((k.replace("smsp__average_warps_issue_stalled_", "").replace("_per_issue_active.ratio", ""),
                      val(d, u, k)) for k in d
                     if k.startswith("smsp__average_warps_issue_stalled_") and k.endswith("_per_issue_active.ratio")),
                    key=lambda x: -x[1])[:3]
        print(f"| {i} | `{name}` | {d.get('launch__grid_size')} | {d.get('launch__registers_per_thread')} | "
              f"{dur * 1e6:.1f} | {rd / 1e6:.1f} | {wr / 1e6:.1f} | {gbps:.0f} | "
              f"{val(d, u, 'sm__inst_issued.avg.pct_of_peak_sustained_active'):.1f} | "
              f"{val(d, u, 'sm__warps_active.avg.pct_of_peak_sustained_active'):.1f} | "
              + ", ".join(f"{k} {v:.2f}" for k, v in st) + " |")


if __name__ == "__main__":
    main(sys.argv[1], sys.argv[2] if len(sys.argv) > 2 else sys.argv[1])
