import sys; sys.path.insert(0, "tests")
import numpy as np, torch
import paper_1911_00357_b200 as dd
import test_gpu_parity as t
ctx = dd.Context(0, 1)
for seed in (1, 2):
    try:
        t._gae_case(dd, ctx, 2, 4, seed)
        print("seed", seed, "ok")
    except AssertionError as e:
        print("seed", seed, "FAIL", str(e)[:300])
