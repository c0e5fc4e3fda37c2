"""Markdown summary of an ncu --set full report: python tools/ncu_summary.py report.ncu-rep"""
import csv
import io
import subprocess
import sys

METRICS = [
    ("gpu__time_duration.sum", "dur"),
    ("dram__bytes_read.sum", "dram_rd"),
    ("dram__bytes_write.sum", "dram_wr"),
    ("gpu__dram_throughput.avg.pct_of_peak_sustained_elapsed", "dram_%"),
    ("sm__pipe_tensor_op_hmma_cycles_active.avg.pct_of_peak_sustained_active", "hmma_%"),
    ("sm__pipe_tensor_cycles_active.avg.pct_of_peak_sustained_active", "tensor_%"),
    ("sm__throughput.avg.pct_of_peak_sustained_elapsed", "sm_%"),
    ("launch__registers_per_thread", "regs"),
    ("launch__grid_size", "grid"),
    ("launch__block_size", "block"),
    ("sm__warps_active.avg.pct_of_peak_sustained_active", "occ_%"),
]


def main(path):
    raw = subprocess.check_output(["ncu", "-i", path, "--page", "raw", "--csv"], stderr=subprocess.DEVNULL).decode()
    rows = list(csv.reader(io.StringIO(raw)))
    hdr, units = rows[0], rows[1]
    idx = {name: hdr.index(name) for name, _ in METRICS if name in hdr}
    ki = hdr.index("Kernel Name")
    print("| kernel | " + " | ".join(short for name, short in METRICS if name in idx) + " |")
    print("|---|" + "---|" * len(idx))
    for r in rows[2:]:
        cells = []
        for name, short in METRICS:
            if name not in idx:
                continue
            v, u = r[idx[name]], units[idx[name]]
            cells.append(f"{v} {u}".strip())
        print(f"| {r[ki].split('(')[0][-40:]} | " + " | ".join(cells) + " |")


if __name__ == "__main__":
    main(sys.argv[1])
