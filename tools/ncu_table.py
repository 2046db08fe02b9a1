"""Markdown table of the roofline-relevant counters of every kernel in one or more ncu --set full reports.
Usage: python tools/ncu_table.py a.ncu-rep [b.ncu-rep ...]"""
import csv
import re
import subprocess
import sys

M = [("gpu__time_duration.sum", "us"), ("dram__bytes_read.sum", "read MB"), ("dram__bytes_write.sum", "write MB"),
     ("smsp__issue_active.avg.pct_of_peak_sustained_active", "issue %"),
     ("sm__warps_active.avg.pct_of_peak_sustained_active", "warps %"),
     ("sm__pipe_fp64_cycles_active.avg.pct_of_peak_sustained_active", "fp64 %"),
     ("sm__pipe_fmaheavy_cycles_active.avg.pct_of_peak_sustained_elapsed", "fmaheavy %"),
     ("sm__inst_executed_pipe_alu.avg.pct_of_peak_sustained_active", "alu %"), ("launch__registers_per_thread", "regs")]
TSCALE = {"ns": 1e-3, "nsecond": 1e-3, "us": 1.0, "usecond": 1.0, "ms": 1e3, "msecond": 1e3}
BSCALE = {"byte": 1e-6, "Kbyte": 1e-3, "Mbyte": 1.0, "Gbyte": 1e3}


def rows(rep):
    out = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
    r = list(csv.reader(out.splitlines()))
    return r[0], r[1], r[2:]


def main(reps):
    print("| kernel | grid | " + " | ".join(lab for _, lab in M) + " | DRAM TB/s | top stalls (per issue) |")
    print("|---|---|" + "---|" * len(M) + "---|---|")
    for rep in reps:
        h, u, rs = rows(rep)
        for r in rs:
            name = r[h.index("Kernel Name")]
            m = re.search(r"::([A-Za-z_0-9]+(<[^>]*>)?)", name)
            d, vals = {}, []
            for k, _ in M:
                try:
                    f = float(r[h.index(k)].replace(",", ""))
                except (ValueError, IndexError):
                    f = None
                unit = u[h.index(k)] if k in h else ""
                if f is not None and k.startswith("gpu__time"):
                    f *= TSCALE.get(unit, 1.0)
                if f is not None and k.startswith("dram__bytes"):
                    f *= BSCALE.get(unit, 1.0)
                d[k] = f
                vals.append("%.1f" % f if f is not None else "-")
            st = []
            for i, k in enumerate(h):
                if "smsp__average_warps_issue_stalled" in k and "per_issue_active" in k:
                    try:
                        st.append((float(r[i].replace(",", "")), k.split("stalled_")[1].split("_per")[0]))
                    except ValueError:
                        pass
            st.sort(reverse=True)
            top = ", ".join("%s %.1f" % (b, a) for a, b in st[:3] if b != "selected")
            t = d["gpu__time_duration.sum"] or 0
            tbs = (d["dram__bytes_read.sum"] + d["dram__bytes_write.sum"]) / t if t else 0.0
            print("| %s | %s | %s | %.2f | %s |" % (m.group(1) if m else name[:40], r[h.index("launch__grid_size")],
                                                    " | ".join(vals), tbs, top))


if __name__ == "__main__":
    main(sys.argv[1:])
