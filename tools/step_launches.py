"""Print the kernels of the last learner step in an ncu launch CSV (name, grid, us)."""
import csv
import sys

rows = list(csv.reader(open(sys.argv[1])))
h = next(i for i, r in enumerate(rows) if r and r[0] == "ID")
hdr = rows[h]
K, V, G, U = hdr.index("Kernel Name"), hdr.index("Metric Value"), hdr.index("Grid Size"), hdr.index("Metric Unit")
data = [r for r in rows[h + 1:] if len(r) > V]
start = max(i for i, r in enumerate(data) if "gae_kernel" in r[K])
pat = sys.argv[2] if len(sys.argv) > 2 else ""
for r in data[start:]:
    if pat in r[K]:
        v = float(r[V].replace(",", "")) / (1000.0 if r[U] == "ns" else 1.0)
        print(f"{v:9.1f} us {r[G]:>16s}  {r[K][:60]}")
