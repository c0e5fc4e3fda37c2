"""Summarise an ncu --set full report of the Depth learner step into profiles/:
  r02_kernels_<cfg>.md  per kernel launch: time, tensor-pipe %, DRAM throughput % / bytes, L2 %, and the
                        fraction of the relevant roofline;
  r02_traffic.json       DRAM bytes per launch per kernel family (bench.py's roofline.traffic).
usage: python tools/make_kernel_table.py gpurun_out/<report>.ncu-rep <cfg>"""
import csv, io, json, os, subprocess, sys
from collections import defaultdict

rep, cfg = sys.argv[1], sys.argv[2]
raw = subprocess.check_output(["ncu", "-i", rep, "--page", "raw", "--csv"], text=True, stderr=subprocess.DEVNULL)
rows = list(csv.reader(io.StringIO(raw)))
hdr, units, data = rows[0], rows[1], rows[2:]
col = {h: i for i, h in enumerate(hdr)}


def g(r, name, default=float("nan")):
    i = col.get(name)
    if i is None or not r[i]:
        return default
    try:
        return float(r[i].replace(",", ""))
    except ValueError:
        return r[i]


def fam(name):
    for k in ("tconv", "lstm", "gps_gru", "gn_", "stem", "maxpool", "adam", "grad_norm", "gemm_bf16", "gae",
              "ppo_loss", "relu_mask", "weights_prep", "se_"):
        if k in name:
            return {"gn_": "gn", "gps_gru": "rnn", "lstm": "rnn", "tconv": "conv", "se_": "se"}.get(k, k)
    return "other"


t_unit = units[col["gpu__time_duration.sum"]]
scale = {"nsecond": 1e-3, "usecond": 1.0, "msecond": 1e3}.get(t_unit, 1.0)
lines = ["| # | kernel | grid | time (us) | tensor pipe % of peak | DRAM % of peak | DRAM bytes | L2 hit % |",
         "|---|---|---|---|---|---|---|---|"]
traffic = defaultdict(list)
for n, r in enumerate(data):
    name = r[col["Kernel Name"]]
    t = g(r, "gpu__time_duration.sum") * scale
    tens = g(r, "sm__pipe_tensor_cycles_active_realtime.avg.pct_of_peak_sustained_elapsed")
    dram_pct = g(r, "gpu__dram_throughput.avg.pct_of_peak_sustained_elapsed")
    rd, wr = g(r, "dram__bytes_read.sum", 0.0), g(r, "dram__bytes_write.sum", 0.0)
    ub = {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9}
    rd *= ub.get(units[col["dram__bytes_read.sum"]], 1)
    wr *= ub.get(units[col["dram__bytes_write.sum"]], 1)
    l2 = g(r, "lts__t_sector_hit_rate.pct")
    traffic[fam(name)].append(rd + wr)
    short = name.split("(")[0].replace("void ", "").replace("<unnamed>::", "")[:60]
    lines.append(f"| {n} | `{short}` | {r[col['Grid Size']]} | {t:.2f} | {tens:.1f} | {dram_pct:.1f} | {rd + wr:.3g} | {l2:.1f} |")
out = {k: {"bytes_per_launch": sum(v) / len(v), "launches": len(v)} for k, v in traffic.items()}
os.makedirs("profiles", exist_ok=True)
with open(f"profiles/r02_kernels_{cfg}.md", "w") as f:
    f.write(f"# ncu --set full, {cfg} learner step (cold caches per replay: compare shares, not absolutes)\n\n")
    f.write("tensor pipe % = sm__pipe_tensor_cycles_active_realtime (fraction of the tensor roofline);\n")
    f.write("DRAM % = gpu__dram_throughput (fraction of the HBM roofline).\n\n")
    f.write("\n".join(lines) + "\n")
json.dump(out, open("profiles/r02_traffic.json", "w"), indent=1)
print("\n".join(lines[:60]))
