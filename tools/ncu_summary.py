"""Summarise an ncu --set full report into a short per-launch table (for profiles/).

    python tools/ncu_summary.py gpurun_out/prof.ncu-rep > profiles/<name>.txt
"""
import csv
import subprocess
import sys

KEYS = [
    ("gpu__time_duration.sum", "us"),
    ("dram__bytes_read.sum", "dram_read"),
    ("dram__bytes_write.sum", "dram_write"),
    ("gpu__dram_throughput.avg.pct_of_peak_sustained_elapsed", "dram_%peak"),
    ("sm__pipe_tensor_cycles_active.avg.pct_of_peak_sustained_elapsed", "tensor_%"),
    ("smsp__issue_active.avg.pct_of_peak_sustained_active", "issue_%"),
    ("sm__warps_active.avg.pct_of_peak_sustained_active", "warps_active_%"),
    ("launch__registers_per_thread", "regs"),
    ("launch__occupancy_limit_shared_mem", "ctas/SM(smem)"),
    ("smsp__inst_executed.sum", "warp_instr"),
]


def main(path):
    out = subprocess.run(["ncu", "-i", path, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
    rows = list(csv.reader(out.splitlines()))
    h, units = rows[0], rows[1]
    for r in rows[2:]:
        name = r[h.index("Kernel Name")].split("(")[0]
        grid = r[h.index("Grid Size")] if "Grid Size" in h else ""
        print(f"{name} grid={grid}")
        for k, label in KEYS:
            if k in h:
                i = h.index(k)
                print(f"    {label:16s} {r[i]} {units[i]}")
        stalls = []
        for i, k in enumerate(h):
            if k.startswith("smsp__average_warps_issue_stalled") and k.endswith("per_issue_active.ratio"):
                try:
                    stalls.append((float(r[i]), k.split("stalled_")[1].split("_per")[0]))
                except ValueError:
                    pass
        top = ", ".join(f"{n} {v:.2f}" for v, n in sorted(stalls, reverse=True)[:4])
        print(f"    top stalls       {top}")


if __name__ == "__main__":
    main(sys.argv[1])
