"""Summarise an ncu --set full report: one row per captured launch."""
import csv
import io
import subprocess
import sys

rep = sys.argv[1]
raw = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
rows = list(csv.reader(io.StringIO(raw)))
hdr, units = rows[0], rows[1]
want = [("Grid Size", "grid"), ("gpu__time_duration.sum", "us"),
        ("dram__bytes_read.sum", "dram_rd"), ("dram__bytes_write.sum", "dram_wr"),
        ("gpu__dram_throughput.avg.pct_of_peak_sustained_elapsed", "dram%"),
        ("sm__pipe_tensor_cycles_active.avg.pct_of_peak_sustained_elapsed", "tensor%"),
        ("lts__throughput.avg.pct_of_peak_sustained_elapsed", "l2%"),
        ("sm__throughput.avg.pct_of_peak_sustained_elapsed", "sm%"),
        ("launch__registers_per_thread", "regs")]
idx = [(hdr.index(k), n, units[hdr.index(k)]) for k, n in want if k in hdr]
print("| # | " + " | ".join(f"{n} ({u})" if u else n for _, n, u in idx) + " |")
print("|" + "---|" * (len(idx) + 1))
for i, r in enumerate(rows[2:]):
    print(f"| {i} | " + " | ".join(r[j] for j, _, _ in idx) + " |")
