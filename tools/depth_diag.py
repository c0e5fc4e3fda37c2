"""Per-tensor relative L2 of the depth network gradients vs the oracle (diagnostic)."""
import sys
import numpy as np
import torch
sys.path.insert(0, "."); sys.path.insert(0, "tests")
import test_gpu_parity as t
import paper_1911_00357_b200 as dd

ctx = dd.Context(0, 1)
E, T, B, lengths = 2, 6, 2, [6, 3]
lay, lg, vl, g, lo, vo, go = t._net_case(dd, ctx, "depth", E, T, B, 40 + E + T, lengths)
print("logits", t.rel_l2(lg, lo), "values", t.rel_l2(vl, vo))
for name, off, shape, _ in lay:
    n = int(np.prod(shape))
    print(f"{name:40s} {t.rel_l2(g[off:off + n], go[off:off + n]):.3e}  |g|={np.linalg.norm(go[off:off+n]):.3e}")
