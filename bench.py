#!/usr/bin/env python
"""DD-PPO learner-step benchmark (BASELINE.json metric: learner experience-steps/sec).

One step = one whole learner step on one rollout per rank (SURVEY.md 8(a) rows a2..a8 + a10):
GAE -> advantage normalisation (allreduce of sum/sum^2) -> 2 epochs x 2 minibatches of
{actor-critic fwd, fused PPO loss+grad, bwd, gradient allreduce + clip + Adam} -> step
accounting allreduce.  Default workload: configs[2] "Depth agent" -- the configuration
BASELINE.json's metric ("at 1/2/4/8 B200") is quoted on: 4 envs/GPU x 128 steps of 64x64 depth,
half-width ResNet18 + GroupNorm + LSTM-512, 2 epochs x 2 minibatches; synthetic PointGoal-shaped
rollouts (synth/), random-init weights.  --config gps|rgbd|stress|toy selects the other configs.

  python bench.py [--gpus N] [--steps K] [--warmup W] [--impl ours|reference] [--config depth]

Multi-GPU: torchrun (one process per GPU, NCCL); weak scaling (E envs per GPU).  The
reference arm (--impl reference) is the CPU oracle (oracle/) run as it stands on the host.
"""
import argparse
import json
import os
import statistics
import subprocess
import sys
import threading
import time

import numpy as np

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

import synth  # noqa: E402

L2_FLUSH_BYTES = 256 << 20  # > 126 MB L2
JSON_OUT = sys.stdout


def parse():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=200)
    ap.add_argument("--warmup", type=int, default=10)
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--config", default="depth", choices=["gps", "toy", "stress_gps", "depth", "rgbd", "stress", "serx50", "serx101",
                                                         "serx101_1024"])
    ap.add_argument("--seed", type=int, default=1337)
    ap.add_argument("--no-e2e", action="store_true")
    ap.add_argument("--e2e-arenas", type=int, default=2, choices=[1, 2],
                    help="device rollout arenas of the e2e loop (2: the H2D copy overlaps the previous step)")
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--conv-engine", default="tma", choices=["tma", "cpasync"],
                    help="visual encoders' convolutions: TMA-fed warp-specialised tcgen05 (default) or the round-1 "
                         "cp.async kernel (A/B)")
    ap.add_argument("--fwd-planes", type=int, default=2, choices=[1, 2],
                    help="encoder forward operands: bf16 hi/lo planes (2, default) or plain bf16 (1)")
    ap.add_argument("--a8", default="auto", choices=["auto", "sharded", "allread"], help="peer-memory a8 form (N > 1)")
    return ap.parse_args()


def dist_env():
    rank = int(os.environ.get("RANK", "0"))
    world = int(os.environ.get("WORLD_SIZE", "1"))
    local = int(os.environ.get("LOCAL_RANK", str(rank)))
    return rank, world, local


# ------------------------------------------------------------------ clocks sampler
class ClockSampler:
    """nvidia-smi sampling of SM clocks and throttle reasons during the timed region."""
    Q = ("index,clocks.sm,clocks.max.sm,power.draw,clocks_event_reasons.active,clocks_event_reasons.hw_slowdown,"
         "clocks_event_reasons.hw_thermal_slowdown,clocks_event_reasons.sw_thermal_slowdown,"
         "clocks_event_reasons.sw_power_cap")

    def __init__(self, device_index):
        self.dev = device_index
        self.proc = None
        self.lines = []

    def start(self):
        try:
            self.proc = subprocess.Popen(["nvidia-smi", "-i", str(self.dev), f"--query-gpu={self.Q}",
                                          "--format=csv,noheader,nounits", "-lms", "100"],
                                         stdout=subprocess.PIPE, stderr=subprocess.DEVNULL, text=True)
            self.thread = threading.Thread(target=self._read, daemon=True)
            self.thread.start()
        except FileNotFoundError:
            self.proc = None

    def _read(self):
        for line in self.proc.stdout:
            self.lines.append(line.strip())

    def stop(self):
        if self.proc is None:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["nvidia-smi unavailable"]}
        time.sleep(0.25)
        self.proc.terminate()
        try:
            self.proc.wait(timeout=5)
        except subprocess.TimeoutExpired:
            self.proc.kill()
        sm, smax, reasons = [], None, set()
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        for ln in self.lines:
            f = [x.strip() for x in ln.split(",")]
            if len(f) < 9:
                continue
            try:
                sm.append(float(f[1]))
                smax = float(f[2])
            except ValueError:
                continue
            for name, val in zip(names, f[5:9]):
                if val.lower() == "active":
                    reasons.add(name)
        return {"sm_mhz": statistics.median(sm) if sm else None, "sm_max_mhz": smax,
                "reasons": sorted(reasons), "samples": len(sm)}


# ------------------------------------------------------------------ reference arm (the CPU oracle)
def cpu_cores():
    try:
        return len(os.sched_getaffinity(0))
    except AttributeError:
        return os.cpu_count()


def blas_threads():
    try:
        from threadpoolctl import threadpool_info
        info = threadpool_info()
        return max([i.get("num_threads", 1) for i in info] or [1])
    except Exception:
        return None


# The oracle's fp64 NumPy ResNet needs ~0.2 s per frame-step of the Depth agent: its bounded sample
# keeps the configuration but shortens the rollouts (whole learner steps on E x ORACLE_T[cfg]).
ORACLE_T = {"depth": 32, "stress": 8, "rgbd": 2, "serx50": 1, "serx101": 1, "serx101_1024": 1}


def oracle_steps_per_sec(cfgname, seed, budget_s=15.0, max_steps=None, T=None):
    """Time the oracle's learner step (oracle/learner.py, as it stands) on the same workload."""
    from oracle import learner as olearner
    from oracle import models
    c = dict(synth.CONFIGS[cfgname])
    c["T"] = T or ORACLE_T.get(cfgname, c["T"])
    offs, P = models.offsets(c["arch"], hidden=c["hidden"])
    fans = {n: f for n, _, f in models.layout(c["arch"], hidden=c["hidden"])}
    p = synth.init_params([(o, int(np.prod(s)), fans[k]) for k, (o, s) in offs.items()], P, seed)
    m = np.zeros(P)
    v = np.zeros(P)
    step, n_steps, exp_steps = 0, 0, 0
    t0 = time.perf_counter()
    it = 0
    while True:
        ro = synth.rollout(c["E"], c["T"], seed, rank=0, iteration=it, hidden=c["hidden"], obs_shape=c.get("obs"),
                           rnn_layers=c.get("rnn_layers", 1))
        pm = synth.perms(seed, it, c["epochs"], c["E"])
        ts = time.perf_counter()
        p, m, v, step, info = olearner.learner_step(c["arch"], p, m, v, step, [ro], [pm],
                                                    dict(epochs=c["epochs"], minibatches=c["minibatches"]),
                                                    hidden=c["hidden"])
        exp_steps += info["steps"]
        n_steps += 1
        it += 1
        el = time.perf_counter() - t0
        if el >= budget_s or (max_steps and n_steps >= max_steps):
            break
        del ts
    return exp_steps / el, n_steps, el


def run_reference(args, rank, world):
    if rank != 0:
        return 0
    c = synth.CONFIGS[args.config]
    # each "step" is one oracle learner step on a bounded sample of the workload (whole rollouts of
    # T_s steps); all of the host's cores (torchrun exports OMP_NUM_THREADS=1 to every rank; rank 0
    # runs alone here)
    try:
        from threadpoolctl import threadpool_limits
        limiter = threadpool_limits(limits=cpu_cores())
    except Exception:
        limiter = None
    T_s = ORACLE_T.get(args.config, c["T"])
    # size the sample so that the K timed steps take about two minutes (probe: one step at T = 2)
    _, _, el1 = oracle_steps_per_sec(args.config, args.seed, budget_s=1e9, max_steps=1, T=2)
    T_s = int(max(2, min(T_s, 2 * 120.0 / (max(args.steps, 1) * max(el1, 1e-3)))))
    for _ in range(args.warmup if args.warmup < 2 else 1):
        oracle_steps_per_sec(args.config, args.seed, budget_s=1e9, max_steps=1, T=T_s)
    sps, n, el = oracle_steps_per_sec(args.config, args.seed, budget_s=1e9, max_steps=args.steps, T=T_s)
    out = {
        "impl": "reference", "metric": "learner experience-steps/sec", "value": sps,
        "unit": "experience-steps/s", "n_gpus": world, "steps": args.steps, "warmup": args.warmup,
        "ms_per_step": 1e3 * el / max(n, 1), "higher_is_better": True, "scaling": "weak", "vs_baseline": None,
        "dtype": "f64", "data": "synthetic",
        "config": {"workload": workload_name(args.config, c), "rank0_only": True,
                   "oracle_sample": f"{c['E']} envs x {T_s} steps per learner step"},
        "cpu_baseline": {"value": sps, "unit": "experience-steps/s", "cores": blas_threads() or cpu_cores(),
                         "kind": "oracle", "sample": f"{n} whole learner steps on {c['E']} envs x {T_s} steps (rank-0 rollout)"},
        "e2e": {"value": sps, "unit": "experience-steps/s", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
    }
    if limiter is not None:
        limiter.restore_original_limits()
    print(json.dumps(out), file=JSON_OUT, flush=True)
    return 0


def workload_name(cfgname, c):
    idx = {"toy": 0, "gps": 1, "stress_gps": 1, "depth": 2, "rgbd": 3, "stress": 4, "serx50": 3, "serx101": 3,
           "serx101_1024": 3}[cfgname]
    net = {"toy": "goal MLP(64, tanh) -> heads",
           "gps": "goal FC + action embedding -> GRU-512 -> heads",
           "depth": "64x64 depth -> ResNet18/2 + GroupNorm -> FC 512; goal FC + action embedding -> LSTM-512 -> heads",
           "serx50": "256x256 RGB-D -> avg-pool -> SE-ResNeXt50/2 (NEXT-3) + GroupNorm -> FC 2048->512; goal FC + "
                     "action embedding -> 2-layer LSTM-512 -> heads",
           "serx101": "256x256 RGB-D -> avg-pool -> SE-ResNeXt101/2 (NEXT-3) + GroupNorm -> FC 2048->512; goal FC + "
                      f"action embedding -> 2-layer LSTM-{c['hidden']} -> heads",
           "rgbd": "256x256 RGB-D -> avg-pool -> ResNet50/2 + GroupNorm -> FC 2048->512; goal FC + action embedding "
                   "-> 2-layer LSTM-512 -> heads"}[c["arch"]]
    return (f"configs[{idx}] {cfgname}: {c['E']} envs/GPU x {c['T']} steps, {net}, "
            f"{c['epochs']} epochs x {c['minibatches']} minibatches, Adam")


# ------------------------------------------------------------------ our arm
def main():
    args = parse()
    # one JSON line on stdout: everything native code prints (NCCL's version banner, warnings) is
    # sent to stderr by pointing fd 1 at fd 2; the JSON line goes to the saved original stdout
    global JSON_OUT
    sys.stdout.flush()
    JSON_OUT = os.fdopen(os.dup(1), "w")
    os.dup2(2, 1)
    rank, world, local = dist_env()
    if args.impl == "reference":
        return run_reference(args, rank, world)

    import torch
    import torch.distributed as dist

    torch.cuda.set_device(local)
    if world > 1:
        dist.init_process_group("nccl", device_id=torch.device("cuda", local))
    import paper_1911_00357_b200 as dd
    from paper_1911_00357_b200.learner import Learner

    uid = None
    if world > 1:
        obj = [dd.get_unique_id() if rank == 0 else None]
        dist.broadcast_object_list(obj, src=0)
        uid = obj[0]
    ctx = dd.Context(rank, world, uid, device=local)
    dd.ddppo_set_conv_engine(ctx, args.conv_engine)
    dd.ddppo_set_fwd_planes(ctx, args.fwd_planes)
    dd.ddppo_set_a8_mode(ctx, args.a8)
    c = synth.CONFIGS[args.config]
    desc = dd.model_desc(c["arch"], c["hidden"])
    lay = dd.param_layout(desc)
    P = dd.param_count(desc)
    p0 = synth.init_params([(off, int(np.prod(s)), fan) for _, off, s, fan in lay], P, args.seed)
    lrn = Learner(ctx, c["arch"], c["E"], c["T"], c["epochs"], c["minibatches"], hidden=c["hidden"], params=p0,
                  normalize_adv=True, rollout_buffers=2)
    stream = torch.cuda.current_stream()
    n_roll = 4  # distinct rollouts cycled through (different data every step)
    preempt = None
    lengths = [None] * n_roll
    if c.get("preempt_p"):
        # configs[4]: each rollout's collection phase under the preemption protocol (untimed, virtual
        # ticks, one NCCL int32 poll per tick); every env of a rank stops at the rank's L_w
        from paper_1911_00357_b200.learner import preempt_collect
        preempt = {"p_percent": c["preempt_p"], "T": c["T"], "rollouts": []}
        K, ms = dd.ddppo_preempt_threshold(dd.preempt_cfg(c["preempt_p"], c["T"]), world)
        preempt.update(K=K, min_steps=ms)
        for i in range(n_roll):
            costs = synth.straggler_costs(args.seed + i, world, c["T"])[rank]
            L_w, ticks = preempt_collect(ctx, costs, c["T"], c["preempt_p"])
            lengths[i] = [L_w] * c["E"]
            cnt = dd.ddppo_allreduce_counts(ctx, [c["E"] * L_w, c["E"] * (c["T"] - L_w), 1 if L_w < c["T"] else 0])
            preempt["rollouts"].append({"ticks": ticks, "collected": int(cnt[0]), "preempted_steps": int(cnt[1]),
                                        "preempted_ranks": int(cnt[2]), "rank0_L": L_w})
    rollouts = [synth.rollout(c["E"], c["T"], args.seed, rank=rank, iteration=i, hidden=desc.hidden,
                              obs_shape=c.get("obs"), length=lengths[i], rnn_layers=c.get("rnn_layers", 1))
                for i in range(n_roll)]
    perms = [synth.perms(args.seed, i, c["epochs"], c["E"], rank=rank) for i in range(n_roll)]
    flush = torch.empty(L2_FLUSH_BYTES // 4, dtype=torch.float32, device="cuda")

    def barrier():
        if world > 1:
            dist.barrier()
        torch.cuda.synchronize()

    # page-locked host arenas, one per rollout: loading one is a single async H2D copy enqueued on the
    # stream ahead of the step (outside its events) -- no host stall, no rank skew from pageable copies
    pinned = []
    for i in range(n_roll):
        hb = lrn.pinned_host_buffers()
        src = lrn.host_fields(rollouts[i])  # frames as bf16 depth (+ uint8 RGB): the rollout's wire format
        for k in hb:
            if k not in ("__arena__", "perms"):
                v = src[k]
                hb[k].copy_((v if isinstance(v, torch.Tensor) else torch.from_numpy(np.ascontiguousarray(v)))
                            .reshape(hb[k].shape))
        pinned.append(hb)

    def step(i):
        lrn.load_rollout(pinned[i % n_roll], perms[i % n_roll], non_blocking=True)
        st = lrn.step(stream)
        counts = dd.ddppo_allreduce_counts(ctx, [lrn.steps_per_rollout()])  # a10 step accounting
        return st, int(counts[0])

    # warm-up
    for i in range(args.warmup):
        step(i)
    barrier()
    ctx.check()

    # ---- device-timed region: inputs already resident in HBM; L2 flushed between steps; the learner
    # step replays its CUDA graph (per-family profiling is off here: it needs per-launch events)
    sampler = ClockSampler(local)
    sampler.start()
    dd.profile_read(ctx, reset=True)
    ev = [(torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)) for _ in range(args.steps)]
    total_exp = 0
    barrier()
    t_wall0 = time.perf_counter()
    for i in range(args.steps):
        lrn.load_rollout(pinned[i % n_roll], perms[i % n_roll], non_blocking=True)  # H2D, outside the events
        flush.zero_()
        ev[i][0].record(stream)
        lrn.step(stream)
        counts = dd.ddppo_allreduce_counts(ctx, [lrn.steps_per_rollout()])  # a10 step accounting
        ev[i][1].record(stream)
        total_exp += int(counts[0])
    barrier()
    t_wall = time.perf_counter() - t_wall0
    launches_timed = dd.profile_read(ctx, reset=True)
    clocks = sampler.stop()
    ctx.check()
    # ---- kernel-family times for the roofline: the same workload again, eager, CUDA events around
    # every family's launches on the launching stream
    prof_steps = min(args.steps, 50)
    dd.profile_enable(ctx, True)
    for i in range(prof_steps):
        lrn.load_rollout(pinned[i % n_roll], perms[i % n_roll], non_blocking=True)
        flush.zero_()
        lrn.step(stream)
        dd.ddppo_allreduce_counts(ctx, [lrn.steps_per_rollout()])
    barrier()
    dd.profile_enable(ctx, False)
    prof = dd.profile_read(ctx, reset=True)
    smem_bytes = dd.profile_smem_bytes(ctx, reset=True)
    dev_ms = sum(a.elapsed_time(b) for a, b in ev)
    t = torch.tensor([dev_ms], dtype=torch.float64, device="cuda")
    if world > 1:
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
    dev_ms = float(t.item())
    value = total_exp / (dev_ms / 1e3)

    # ---- end-to-end: host (pinned) rollout -> device each step, stats read back each step
    e2e = None
    if not args.no_e2e:
        # (the same packed pinned arenas: one H2D copy per step, inside this timed region)
        h2d = pinned[0]["__arena__"].numel()
        d2h = lrn.stats.numel() * 4
        # a training loop's shape: step i+1 is enqueued before step i's statistics are read back (two
        # statistics buffers, D2H on a copy stream after step i's completion event); the rollout H2D
        # copies run on their own stream into the arena the previous step is not reading (two device
        # arenas), so step i+1's input transfer overlaps step i
        stats_dev = [torch.zeros_like(lrn.stats) for _ in range(2)]
        stats_host = [torch.zeros(lrn.stats.shape, dtype=lrn.stats.dtype).pin_memory() for _ in range(2)]
        copy_stream = torch.cuda.Stream()
        h2d_stream = torch.cuda.Stream()
        done = [torch.cuda.Event() for _ in range(2)]
        h2d_st = h2d_stream if args.e2e_arenas == 2 else None
        for i in range(4):  # warm the loop's own buffers and graph keys (2 arenas x 2 uses; not timed)
            lrn.load_rollout(pinned[i % n_roll], perms[i % n_roll], non_blocking=True, copy_stream=h2d_st)
            lrn.step(stream, stats=stats_dev[i % 2])
            dd.ddppo_allreduce_counts(ctx, [lrn.steps_per_rollout()])
        barrier()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e_exp = 0
        e0.record(stream)
        for i in range(args.steps):
            lrn.load_rollout(pinned[i % n_roll], perms[i % n_roll], non_blocking=True, copy_stream=h2d_st)
            lrn.step(stream, stats=stats_dev[i % 2])
            copy_stream.wait_stream(stream)
            with torch.cuda.stream(copy_stream):
                stats_host[i % 2].copy_(stats_dev[i % 2], non_blocking=True)  # D2H of the step's loss statistics
                done[i % 2].record(copy_stream)
            if i > 0:
                done[(i - 1) % 2].synchronize()  # step i-1's result is on the host
            counts = dd.ddppo_allreduce_counts(ctx, [lrn.steps_per_rollout()])
            e_exp += int(counts[0])
        done[(args.steps - 1) % 2].synchronize()
        e1.record(stream)
        barrier()
        e_ms = torch.tensor([e0.elapsed_time(e1)], dtype=torch.float64, device="cuda")
        if world > 1:
            dist.all_reduce(e_ms, op=dist.ReduceOp.MAX)
        e2e = {"value": e_exp / (float(e_ms.item()) / 1e3), "unit": "experience-steps/s",
               "h2d_bytes_per_step": int(h2d), "d2h_bytes_per_step": int(d2h)}

    # ---- roofline of the dominant kernel family (device time measured live above)
    peaks = {}
    try:
        peaks = json.load(open(os.path.join(ROOT, "MEASURED_PEAKS.json")))
    except Exception:
        pass
    fam_ms = {k: v[0] for k, v in prof.items()}
    # the dominant kernel: the TMA implicit-GEMM convolution for the visual agents, the GRU
    # recurrence for GPS (sub-families "conv" / "rnn": CUDA events around each launch on its stream)
    dom = "conv" if c["arch"] in ("depth", "rgbd", "serx50", "serx101") else "rnn" if c["arch"] == "gps" else "net_fwd"
    launches = {k: v[1] for k, v in launches_timed.items()}
    roofline = roofline_for(dom, prof, c, lrn, peaks, prof_steps, smem_bytes)
    kernels = kernel_table(prof, c, lrn, peaks, prof_steps)
    gpu_launches = int(sum(v for k, v in launches.items() if k != "allreduce"))

    cpu_base = None
    if rank == 0 and world == 1 and not args.no_cpu_baseline:
        sps, n, el = oracle_steps_per_sec(args.config, args.seed, budget_s=12.0)
        T_s = ORACLE_T.get(args.config, c["T"])
        cpu_base = {"value": sps, "unit": "experience-steps/s", "cores": blas_threads() or cpu_cores(),
                    "kind": "oracle",
                    "sample": f"{n} whole learner steps on {c['E']} envs x {T_s} steps of this config ({el:.1f} s)"}

    if rank == 0:
        out = {
            "metric": "learner experience-steps/sec", "value": value, "unit": "experience-steps/s",
            "n_gpus": world, "steps": args.steps, "warmup": args.warmup,
            "ms_per_step": dev_ms / args.steps, "higher_is_better": True, "scaling": "weak",
            "vs_baseline": None, "dtype": "f32+f16/bf16-mma", "data": "synthetic",
            "config": {"workload": workload_name(args.config, c),
                       "E_per_gpu": c["E"], "T": c["T"], "params": P, "parallelism": f"dp{world}",
                       "l2": "flushed between timed steps (256 MiB write), per-step CUDA events",
                       "wall_s_timed_loop": t_wall},
            "clocks": clocks, "e2e": e2e, "gpu_launches": gpu_launches, "preemption": preempt,
            "kernel_ms": {k: round(v, 4) for k, v in fam_ms.items() if v > 0},
            "kernel_ms_steps": prof_steps, "kernels": kernels,
            "roofline": roofline, "cpu_baseline": cpu_base,
        }
        print(json.dumps(out), file=JSON_OUT, flush=True)
    if world > 1:
        dist.barrier()
        dist.destroy_process_group()
    ctx.close()
    return 0


def depth_encoder_macs(arch="depth"):
    """Multiply-accumulates per frame of the visual agents' encoders (depth: 64x64 -> ResNet18/2 ->
    128x2x2; rgbd: 256x256 -> avg-pool -> ResNet50/2 -> 128x4x4)."""
    macs = 0

    def conv(h, ci, co, k, s, p):
        nonlocal macs
        ho = (h + 2 * p - k) // s + 1
        macs += ho * ho * co * ci * k * k
        return ho
    rgbd = arch == "rgbd"
    h = conv(128 if rgbd else 64, 4 if rgbd else 1, 32, 7, 2, 3)
    stem = macs
    h = (h + 2 - 3) // 2 + 1  # max-pool
    cin = 32
    for li, w in enumerate((32, 64, 128, 256)):
        for bi in range((3, 4, 6, 3)[li] if rgbd else 2):
            s = 2 if (bi == 0 and li > 0) else 1
            cout = 4 * w if rgbd else w
            if rgbd:
                conv(h, cin, w, 1, 1, 0)
                h1 = conv(h, w, w, 3, s, 1)
                conv(h1, w, cout, 1, 1, 0)
            else:
                h1 = conv(h, cin, w, 3, s, 1)
                conv(h1, w, w, 3, 1, 1)
            if s != 1 or cin != cout:
                conv(h, cin, cout, 1, s, 0)
            h, cin = h1, cout
    conv(h, cin, 128, 3, 1, 1)
    return {"all": macs, "stem": stem}


def _traffic(*kernels):
    """DRAM bytes per launch of a kernel from the committed ncu --set full capture summary
    (profiles/r01_traffic.json, tools/make_traffic.py); None if it was not captured."""
    try:
        t = json.load(open(os.path.join(os.path.dirname(os.path.abspath(__file__)), "profiles", "r01_traffic.json")))
    except (OSError, ValueError):
        return None
    vals = [t[k]["bytes_per_launch"] for k in kernels if k in t]
    return sum(vals) if len(vals) == len(kernels) else None


def _traffic_r02(kind):
    """DRAM bytes per launch of a kernel kind from the committed ncu --set full capture summary
    (profiles/r02_traffic.json, written by tools/make_traffic.py); None if not captured."""
    try:
        t = json.load(open(os.path.join(ROOT, "profiles", "r02_traffic.json")))
    except (OSError, ValueError):
        return None
    return t.get(kind, {}).get("bytes_per_launch")


def roofline_for(fam, prof, c, lrn, peaks, steps, smem_bytes=None):
    """The dominant kernel: its algorithmic work (host-side accounting at each launch: useful dense
    FLOPs, the bf16x3 forward counted once) / its device time (CUDA events around every launch on
    the launching stream, the eager profiling pass), against the measured sustained bf16 peak."""
    ms, n, flops = prof[fam]
    bf16 = peaks.get("bf16_tflops_sustained", 1400.0)
    per_launch_s = (ms / 1e3) / max(n, 1)
    achieved = flops / max(ms / 1e3, 1e-12) / 1e12
    kern = {"conv": "tconv_kernel (TMA implicit-GEMM FPROP / DGRAD / WGRAD)",
            "rnn": "gps_gru_fwd/bwd_kernel" if c["arch"] == "gps" else
            "lstm1024_fwd/bwd_kernel" if c["hidden"] == 1024 else "lstm_fwd/bwd_kernel"}.get(fam, fam)
    out = {"bound": "tensor", "kernel": kern, "achieved": achieved, "peak": bf16, "unit": "TFLOP/s",
           "frac": achieved / bf16, "traffic": _traffic_r02(fam), "launch_us": per_launch_s * 1e6,
           "launches_per_step": n / max(steps, 1), "flops_per_launch": flops / max(n, 1),
           "share_of_step": ms / max(sum(v[0] for k, v in prof.items() if k in (
               "gae", "adv_norm", "net_fwd", "head", "loss", "net_bwd", "wgrad", "allreduce", "adam", "other")), 1e-9)}
    if smem_bytes and smem_bytes.get(fam, 0) > 0:
        # the binding resource of the conv kernels for N <= 64: shared-memory traffic
        # (TMA operand writes + the bf16x3 MMAs' operand reads) against 128 B / cycle / SM at the max
        # SM clock over the whole chip (side-stream launches use a quarter of the SMs: a lower bound)
        sm_peak = 148 * 128 * peaks.get("sm_max_mhz", 1965.0) * 1e6 / 1e12
        sm_ach = smem_bytes[fam] / max(ms / 1e3, 1e-12) / 1e12
        out["smem"] = {"achieved": sm_ach, "peak": sm_peak, "unit": "TB/s", "frac": sm_ach / sm_peak,
                       "bytes_per_launch": smem_bytes[fam] / max(n, 1)}
    if fam == "rnn":
        out["note"] = ("latency-bound dependency chain (B = E/2 envs x 128 steps on one 16-CTA cluster); "
                       "per-step phases in DESIGN.md")
    else:
        out["note"] = ("small implicit GEMMs (N = 32..256, <= 512 tiles): shared-memory-bandwidth bound for "
                       "N <= 64 ('smem'), per-kernel table in 'kernels' and profiles/r02_kernels_depth.md")
    return out


def kernel_table(prof, c, lrn, peaks, steps):
    """Per kernel (sub-)family: ms and launches per step, achieved rate and fraction of its roofline
    (tensor: measured sustained bf16; HBM: measured copy bandwidth)."""
    hbm = peaks.get("hbm_gbs", 6650.0)
    bf16 = peaks.get("bf16_tflops_sustained", 1400.0)
    E, T = c["E"], c["T"]
    B = E // c["minibatches"]
    out = {}
    for fam, (ms, n, flops) in prof.items():
        if ms <= 0:
            continue
        row = {"ms_per_step": ms / max(steps, 1), "launches_per_step": n / max(steps, 1)}
        if flops > 0:
            a = flops / (ms / 1e3) / 1e12
            row.update(achieved_tflops=a, frac=a / bf16)
        # algorithmic bytes per step: GAE 17 B per element (once per step); loss 60 B per sample and
        # Adam 28 B per parameter (read g, p, m, v; write p, m, v) once per minibatch update
        n_mb = c["epochs"] * c["minibatches"]
        byts = {"gae": 17.0 * E * T, "loss": 60.0 * B * T * n_mb, "adam": 28.0 * lrn.P * n_mb}.get(fam)
        if byts:
            a = byts * steps / (ms / 1e3) / 1e9
            row.update(achieved_gbs=a, frac=a / hbm)
        out[fam] = row
    return out


if __name__ == "__main__":
    sys.exit(main())
