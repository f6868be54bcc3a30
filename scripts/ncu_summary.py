"""Compact per-kernel summary of an ncu report (run here, no GPU needed).

    python scripts/ncu_summary.py gpurun_out/x_full.ncu-rep > profiles/x_summary.md
"""
import csv
import io
import subprocess
import sys

METRICS = [
    ("time_ms", "gpu__time_duration.sum", "ms"),
    ("dram_rd_GB", "dram__bytes_read.sum", "GB"),
    ("dram_wr_GB", "dram__bytes_write.sum", "GB"),
    ("dram_%peak", "dram__throughput.avg.pct_of_peak_sustained_elapsed", None),
    ("tensor_%", "sm__pipe_tensor_cycles_active.avg.pct_of_peak_sustained_active", None),
    ("tc_inst_%", "sm__inst_executed_pipe_tc.avg.pct_of_peak_sustained_active", None),
    ("hmma_%", "sm__inst_executed_pipe_tensor_subpipe_hmma.avg.pct_of_peak_sustained_active", None),
    ("sm_thru_%", "sm__throughput.avg.pct_of_peak_sustained_elapsed", None),
    ("l2_%", "lts__t_sectors.avg.pct_of_peak_sustained_elapsed", None),
    ("l2_hit_%", "lts__t_sector_hit_rate.pct", None),
    ("regs", "launch__registers_per_thread", None),
    ("occ_%", "sm__warps_active.avg.pct_of_peak_sustained_active", None),
    ("sm_MHz", "sm__cycles_elapsed.avg.per_second", "MHz"),
]
SCALE = {("ms", "ns"): 1e-6, ("ms", "us"): 1e-3, ("ms", "usecond"): 1e-3, ("ms", "msecond"): 1.0,
         ("ms", "nsecond"): 1e-6, ("ms", "ms"): 1.0, ("GB", "byte"): 1e-9, ("GB", "Kbyte"): 1e-6,
         ("GB", "Mbyte"): 1e-3, ("GB", "Gbyte"): 1.0, ("GB", "Tbyte"): 1e3, ("MHz", "hz"): 1e-6,
         ("MHz", "Khz"): 1e-3, ("MHz", "Mhz"): 1.0, ("MHz", "Ghz"): 1e3, ("MHz", "cycle/second"): 1e-6,
         ("MHz", "cycle/nsecond"): 1e3, ("MHz", "cycle/usecond"): 1.0}


def main(path):
    raw = subprocess.run(["ncu", "-i", path, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
    rows = list(csv.reader(io.StringIO(raw)))
    hdr, units = rows[0], rows[1]
    col = {h: i for i, h in enumerate(hdr)}
    print("| kernel | " + " | ".join(m[0] for m in METRICS) + " |")
    print("|" + "---|" * (len(METRICS) + 1))
    for r in rows[2:]:
        name = r[col["Kernel Name"]].split("(")[0].replace("void ", "")[:48]
        cells = []
        for label, metric, want in METRICS:
            i = col.get(metric)
            if i is None or not r[i]:
                cells.append("-")
                continue
            try:
                v = float(r[i].replace(",", ""))
            except ValueError:
                cells.append(r[i])
                continue
            if want:
                v *= SCALE.get((want, units[i]), float("nan"))
            cells.append(f"{v:.4g}")
        print(f"| {name} | " + " | ".join(cells) + " |")


if __name__ == "__main__":
    main(sys.argv[1])
