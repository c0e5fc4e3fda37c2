"""Single-plane (bf16) vs hi/lo (bf16x3) encoder forward: parity against the oracle for the Depth network
at the config minibatch (F = 256) -- the largest adopted-decision ratio |pre| / rms and the worst
per-tensor gradient error -- plus the relative time (tools/, a measurement probe)."""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np, torch
import paper_1911_00357_b200 as dd
from tests import test_gpu_parity as tp

ctx = dd.Context(0, 1)
for planes in (2, 1):
    dd.ddppo_set_fwd_planes(ctx, planes)
    for tie in (2.5e-4, 1e-3, 4e-3, 1.6e-2):
        orig = tp._adopt_decisions.__defaults__
        tp._adopt_decisions.__defaults__ = (tie,)
        try:
            lay, lg, vl, g, lo, vo, go = tp._net_case(dd, ctx, "depth", 4, 128, 2, 77)
            worst = max(tp.rel_l2(g[off:off + int(np.prod(s))], go[off:off + int(np.prod(s))]) for _, off, s, _ in lay)
            print(f"planes {planes} tie {tie:g}: ok; logits {tp.rel_l2(lg, lo):.2e} values {tp.rel_l2(vl, vo):.2e} "
                  f"worst grad {worst:.2e}", flush=True)
            break
        except AssertionError as e:
            print(f"planes {planes} tie {tie:g}: {str(e)[:120]}", flush=True)
        finally:
            tp._adopt_decisions.__defaults__ = orig
