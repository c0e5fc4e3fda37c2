"""HBM-roofline microbenchmarks of the memory-bound kernels (GAE scan, PPO loss, clip+Adam) at
sizes far above L2, through the C ABI.  Algorithmic bytes per unit:
  GAE   17 B / element   (r 4 + V 4 + done 1 + A 4 + R 4)
  loss  60 B / sample    (logits 16 + value 4 + action 4 + lp_old 4 + V_old 4 + R 4 + A 4; dlogits 16 + dv 4)
  Adam  28 B / parameter algorithmic (g, p, m, v read 16 + p, m, v write 12; the norm pass's second
        read of g is not counted)
Prints one JSON line per kernel.  Usage: python tools/microbench.py [--reps 10]
"""
import argparse
import json
import os
import sys

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_1911_00357_b200 as dd  # noqa: E402


def timed(fn, reps, flush):
    for _ in range(3):
        fn()
    ts = []
    for _ in range(reps):
        flush.zero_()
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        a.record()
        fn()
        b.record()
        torch.cuda.synchronize()
        ts.append(a.elapsed_time(b) / 1e3)
    return float(np.median(ts))


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--reps", type=int, default=10)
    args = ap.parse_args()
    peaks = json.load(open(os.path.join(os.path.dirname(os.path.dirname(os.path.abspath(__file__))),
                                        "MEASURED_PEAKS.json")))
    hbm = peaks["hbm_gbs"]
    ctx = dd.Context(0, 1)
    flush = torch.empty(256 << 18, dtype=torch.float32, device="cuda")
    g = torch.Generator(device="cuda").manual_seed(0)
    out = []
    # ---- GAE: E = 2^20 envs x T = 128
    E, T, ld = 1 << 20, 128, 132
    rew = torch.randn(E, ld, device="cuda", generator=g)
    val = torch.randn(E, ld, device="cuda", generator=g)
    done = (torch.rand(E, ld, device="cuda", generator=g) < 0.02).to(torch.uint8)
    length = torch.full((E,), T, dtype=torch.int32, device="cuda")
    adv = torch.empty(E, ld, device="cuda")
    ret = torch.empty(E, ld, device="cuda")
    st = torch.zeros(3, dtype=torch.float64, device="cuda")
    s = timed(lambda: dd.ddppo_gae(ctx, rew, val, done, length, E, T, ld, 0.99, 0.95, adv, ret, st), args.reps, flush)
    b = 17.0 * E * T
    out.append(dict(kernel="gae_scan", units=E * T, unit="element", algorithmic_bytes=b, seconds=s,
                    achieved_gbs=b / s / 1e9, peak_gbs=hbm, frac=b / s / 1e9 / hbm))
    del rew, val, done, adv, ret
    # ---- loss: M = 2^24 samples (B = 2^17 envs x 128)
    Bn, T = 1 << 17, 128
    M = Bn * T
    ld = 132
    logits = torch.randn(M, 4, device="cuda", generator=g)
    values = torch.randn(M, device="cuda", generator=g)
    action = torch.randint(0, 4, (Bn, ld), dtype=torch.int32, device="cuda", generator=g)
    lpo = torch.log(torch.rand(Bn, ld, device="cuda", generator=g) * 0.9 + 0.05)
    vo = torch.randn(Bn, ld, device="cuda", generator=g)
    rr = torch.randn(Bn, ld, device="cuda", generator=g)
    aa = torch.randn(Bn, ld, device="cuda", generator=g)
    env_idx = torch.arange(Bn, dtype=torch.int32, device="cuda")
    length = torch.full((Bn,), T, dtype=torch.int32, device="cuda")
    goal = torch.zeros(Bn, T, 3, device="cuda")
    batch = dd.make_batch(goal, None, None, None, length, env_idx, Bn, T, ld, Bn, T, M)
    dl = torch.empty(M, 4, device="cuda")
    dv = torch.empty(M, device="cuda")
    stats = torch.zeros(8, device="cuda")
    mis = torch.tensor([0.1, 1.2], device="cuda")
    cfg = dd.loss_cfg()
    s = timed(lambda: dd.ddppo_ppo_loss_grad(ctx, logits, values, batch, action, lpo, vo, rr, aa, mis, cfg, dl, dv,
                                             stats), args.reps, flush)
    b = 60.0 * M
    out.append(dict(kernel="ppo_loss_grad", units=M, unit="sample", algorithmic_bytes=b, seconds=s,
                    achieved_gbs=b / s / 1e9, peak_gbs=hbm, frac=b / s / 1e9 / hbm))
    del logits, values, action, lpo, vo, rr, aa, dl, dv
    # ---- clip + Adam: P = 64 M parameters (N = 1: no allreduce)
    P = 1 << 26
    grad = torch.randn(P, device="cuda", generator=g) * 1e-3
    prm = torch.randn(P, device="cuda", generator=g)
    m = torch.zeros(P, device="cuda")
    v = torch.zeros(P, device="cuda")
    step = [0]

    def adam():
        step[0] += 1
        dd.ddppo_grad_allreduce_step(ctx, grad, prm, m, v, dd.adam_cfg(step[0]))
    s = timed(adam, args.reps, flush)
    b = 28.0 * P
    out.append(dict(kernel="clip_adam", units=P, unit="parameter", algorithmic_bytes=b, seconds=s,
                    achieved_gbs=b / s / 1e9, peak_gbs=hbm, frac=b / s / 1e9 / hbm))
    ctx.check()
    for o in out:
        print(json.dumps(o))


if __name__ == "__main__":
    main()
