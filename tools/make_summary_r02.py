"""Regenerate profiles/r02_summary.md from the committed round-2 artefacts (run from the repo root)."""
import glob, json, os, subprocess


def ld(p):
    return json.loads(open(p).read().strip().splitlines()[-1])


def line(name, p):
    d = ld(p)
    r = d.get("roofline") or {}
    e2e = (d.get("e2e") or {}).get("value")
    roof = (f"{r.get('kernel')}: {r.get('achieved', 0):.2f} {r.get('unit')} = {100 * r.get('frac', 0):.2f} % of "
            f"{r.get('peak'):.1f} ({r.get('bound')})") if r else ""
    clk = d.get("clocks") or {}
    return (f"| {name} | {d.get('n_gpus', 1)} | {d['value']:.0f} | {d['ms_per_step']:.3f} | "
            f"{e2e:.0f} | {roof} | {clk.get('sm_mhz', '')} / {clk.get('sm_max_mhz', '')} {clk.get('reasons', '')} |"
            if e2e is not None else
            f"| {name} | {d.get('n_gpus', 1)} | {d['value']:.0f} | {d['ms_per_step']:.3f} | -- | {roof} | |")


rows = []
for name, p in [("depth (configs[2], the metric's config)", "profiles/r02_bench_depth.json"),
                ("gps (configs[1])", "profiles/r02_bench_gps.json"),
                ("rgbd (configs[3])", "profiles/r02_bench_rgbd.json"),
                ("serx50 (NEXT-3)", "profiles/r02_bench_serx50.json"),
                ("serx101 (NEXT-3)", "profiles/r02_bench_serx101.json"),
                ("serx101_1024 (NEXT-3: SE-ResNeXt101 + LSTM-1024)", "profiles/r02_bench_serx101_1024.json")]:
    if os.path.exists(p):
        rows.append(line(name, p))
scale = []
for cfg in ("depth", "gps", "stress"):
    for n, tag in ((1, "2-GPU box"), (2, "2-GPU box"), ("1_box4", "4-GPU box"), (4, "4-GPU box")):
        p = f"profiles/r02_scale_{cfg}_n{n}.json"
        if os.path.exists(p):
            scale.append(line(f"{cfg} ({tag})", p))
ref = ld("profiles/r02_reference_depth.json") if os.path.exists("profiles/r02_reference_depth.json") else None
kt = open("profiles/r02_kernels_depth.md").read().split("## First 80 launches")[0].split("## Top kernels by captured time")[1]
floor = open("profiles/r02_rnn_floor.txt").read()
gaps = open("profiles/r02_gaps.txt").read() if os.path.exists("profiles/r02_gaps.txt") else ""
launches = ""
if os.path.exists("profiles/r02_launches_depth.csv"):
    launches = subprocess.check_output(["python", "tools/launches.py", "profiles/r02_launches_depth.csv"]).decode()
kp = {c: open(f"profiles/r02_kprof_{c}.txt").read().splitlines() for c in ("depth", "gps", "rgbd")
      if os.path.exists(f"profiles/r02_kprof_{c}.txt")}
out = f"""# Round 2 profiles (B200, sm_100a, driver 580.159, CUDA 12.9)

Bench numbers come from `bench.py` (CUDA events on the launching stream, max over ranks, L2 flushed
between steps, no profiler).  ncu captures: one GPU, `--clock-control none`, serialised cold-cache
replays (compare shares, not absolutes).  `r02_kprof_*.txt`: CUPTI per-kernel device times of warm,
graph-replayed learner steps (`tools/kprof.py`, taken with `DDPPO_PDL=0`: with programmatic dependent
launch a kernel's CUPTI duration includes its early-launched CTAs' wait).  Regenerate this file with
`python tools/make_summary_r02.py`.

## Bench lines, one GPU

| config | GPUs | value (exp-steps/s) | ms/step | e2e (host buffers) | roofline (dominant kernel) | clocks MHz |
|---|---|---|---|---|---|---|
""" + "\n".join(rows) + """

## Weak scaling (one box, NVLink peer-memory a8)

| config | GPUs | value (exp-steps/s) | ms/step | e2e | roofline | clocks |
|---|---|---|---|---|---|---|
""" + "\n".join(scale) + f"""

## Reference arm (the CPU oracle, `bench.py --impl reference`)

{json.dumps(ref) if ref else "(not run)"}

## Per-kernel table, Depth learner step (`r02_kernels_depth.md`)
{kt}
## Recurrence floor (`r02_rnn_floor.txt`, `tools/rnn_floor.cu`)

```
{floor.strip()}
```

## Gaps between kernels (`r02_gaps.txt`, `tools/gaps.py`)

```
{gaps.strip()}
```

## Launch list of the bench command (`r02_launches_depth.csv`)

`ncu --metrics gpu__time_duration.sum --clock-control none --csv python bench.py --steps 2 --warmup 3 --no-e2e --no-cpu-baseline`

```
{launches.strip()}
```
"""
for c, l in kp.items():
    out += f"\n## CUPTI per-kernel split, {c} (`r02_kprof_{c}.txt`)\n\n```\n" + "\n".join(l[:26]) + "\n```\n"
open("profiles/r02_summary.md", "w").write(out)
print("wrote profiles/r02_summary.md")
