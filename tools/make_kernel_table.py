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
for i, h in enumerate(hdr):  # section-prefixed raw names ("TPC.TriageCompute.<metric>") by their suffix
    base = h.split(".", 2)[-1] if h.count(".") >= 2 and h.split(".")[0].isupper() else h
    col.setdefault(base, i)
    if "." in h:
        col.setdefault(h[h.find(".") + 1:], i)
        col.setdefault(h[h.find(".", h.find(".") + 1) + 1:], i)


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
ub = {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9}
lines = ["| # | kernel | grid | time (us) | tensor pipe % of peak | DRAM % of peak | DRAM bytes | L2 hit % |",
         "|---|---|---|---|---|---|---|---|"]
traffic = defaultdict(list)
agg = defaultdict(lambda: [0, 0.0, 0.0, 0.0, 0.0, 0.0])  # launches, time, tensor%*t, dram%*t, bytes, l2*t
for n, r in enumerate(data):
    name = r[col["Kernel Name"]]
    t = g(r, "gpu__time_duration.sum") * scale
    tens = g(r, "sm__pipe_tensor_cycles_active.avg.pct_of_peak_sustained_active")
    if not isinstance(tens, float) or tens != tens:
        tens = g(r, "sm__pipe_tensor_cycles_active_realtime.avg.pct_of_peak_sustained_elapsed")
    if not isinstance(tens, float):
        tens = float("nan")
    dram_pct = g(r, "gpu__dram_throughput.avg.pct_of_peak_sustained_elapsed")
    rd, wr = g(r, "dram__bytes_read.sum", 0.0), g(r, "dram__bytes_write.sum", 0.0)
    rd *= ub.get(units[col["dram__bytes_read.sum"]], 1)
    wr *= ub.get(units[col["dram__bytes_write.sum"]], 1)
    l2 = g(r, "lts__t_sector_hit_rate.pct")
    traffic[fam(name)].append(rd + wr)
    short = name.split("(")[0].replace("void ", "").replace("<unnamed>::", "")[:60]
    a = agg[short]
    a[0] += 1; a[1] += t; a[2] += tens * t; a[3] += dram_pct * t; a[4] += rd + wr; a[5] += l2 * t
    if n < 80:
        lines.append(f"| {n} | `{short}` | {r[col['Grid Size']]} | {t:.2f} | {tens:.1f} | {dram_pct:.1f} | {rd + wr:.3g} | {l2:.1f} |")
tot = sum(a[1] for a in agg.values())
top = ["| kernel | launches | share of captured time | mean time (us) | tensor pipe % (time-weighted) | DRAM % (time-weighted) | DRAM bytes / launch | L2 hit % |",
       "|---|---|---|---|---|---|---|---|"]
for short, a in sorted(agg.items(), key=lambda kv: -kv[1][1])[:12]:
    top.append(f"| `{short}` | {a[0]} | {100 * a[1] / tot:.1f} % | {a[1] / a[0]:.2f} | {a[2] / a[1]:.1f} | "
               f"{a[3] / a[1]:.1f} | {a[4] / a[0]:.3g} | {a[5] / a[1]:.1f} |")
out = {k: {"bytes_per_launch": sum(v) / len(v), "launches": len(v)} for k, v in traffic.items()}
os.makedirs("profiles", exist_ok=True)
with open(f"profiles/r02_kernels_{cfg}.md", "w") as f:
    f.write(f"# ncu (sections SpeedOfLight, ComputeWorkloadAnalysis, MemoryWorkloadAnalysis + DRAM bytes + tensor pipe), {cfg} learner step ({len(data)} launches captured; ncu replays each launch with\n"
            "# cold caches and serialised: compare shares, not absolute times)\n\n")
    f.write("tensor pipe % = sm__pipe_tensor_cycles_active.avg.pct_of_peak_sustained_active (tensor-pipe busy "
            "cycles over the active SMs' cycles);\n"
            "DRAM % = gpu__dram_throughput (fraction of the HBM roofline).\n\n")
    f.write("## Top kernels by captured time\n\n" + "\n".join(top) + "\n\n")
    f.write("## First 80 launches\n\n" + "\n".join(lines) + "\n")
json.dump(out, open("profiles/r02_traffic.json", "w"), indent=1)
print("\n".join(top))
