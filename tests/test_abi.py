"""CPU checks of the C ABI: the library loads, exports every declared symbol, and its host-side
arithmetic (layouts, preemption thresholds/decisions) agrees with the oracle.  No GPU calls."""
import os
import re
import subprocess

import numpy as np
import pytest

import paper_1911_00357_b200 as dd
from oracle import models, preempt

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def _declared():
    src = open(os.path.join(ROOT, "include", "ddppo.h")).read()
    src = re.sub(r"/\*.*?\*/", "", src, flags=re.S)  # drop comments
    return sorted(set(re.findall(r"^[ \t]*(?:[\w*]+[ \t]+)+\**(ddppo_\w+)[ \t]*\(", src, re.M)))


def test_every_declared_symbol_is_exported():
    names = _declared()
    assert len(names) >= 20
    out = subprocess.check_output(["nm", "-D", "--defined-only", dd._lib.LIB_PATH]).decode()
    exported = set(re.findall(r" T (ddppo_\w+)", out))
    missing = [n for n in names if n not in exported]
    assert not missing, missing
    assert set(dd._lib.EXPORTS) == set(names)
    assert dd.lib.ddppo_abi_version() == 1


def test_library_is_sm100a():
    out = subprocess.check_output(["cuobjdump", "--list-elf", dd._lib.LIB_PATH]).decode()
    assert "sm_100a" in out


@pytest.mark.parametrize("arch,hidden", [("toy", None), ("gps", None), ("depth", None), ("rgbd", None),
                                         ("serx50", None), ("serx101", None),
                                         ("depth", 1024), ("serx101", 1024)])  # NEXT-3's 1024-d LSTM
def test_layout_matches_oracle(arch, hidden):
    kw = {} if hidden is None else {"hidden": hidden}
    lay = dd.param_layout(dd.model_desc(arch, hidden))
    offs, P = models.offsets(arch, **kw)
    assert dd.param_count(dd.model_desc(arch, hidden)) == P
    ref = models.layout(arch, **kw)
    assert [n for n, *_ in lay] == [n for n, _, _ in ref]
    for (name, off, shape, fan), (rname, rshape, rfan) in zip(lay, ref):
        assert off == offs[name][0] and tuple(shape) == tuple(rshape) and fan == rfan


def test_bad_descriptor_rejected():
    with pytest.raises(dd.DdppoError):
        dd.param_count(dd.model_desc("gps", hidden=256))
    with pytest.raises(dd.DdppoError):  # the GRU agent is built for 512 only
        dd.param_count(dd.model_desc("gps", hidden=1024))
    with pytest.raises(dd.DdppoError):
        dd.param_count(dd.model_desc("depth", hidden=768))


def test_preempt_threshold_and_decide_match_oracle():
    for N in (1, 2, 3, 4, 5, 8, 64):
        for p in (1, 10, 50, 60, 80, 100):
            for ow in (False, True):
                for T in (4, 5, 128):
                    K, ms = dd.ddppo_preempt_threshold(dd.preempt_cfg(p, T, other_workers=ow), N)
                    assert K == preempt.threshold_count(p, N, ow)
                    assert ms == preempt.min_steps(T)
    cfg = dd.preempt_cfg(60, 128)
    rng = np.random.default_rng(0)
    for _ in range(2000):
        s, f = int(rng.integers(0, 129)), int(rng.integers(0, 5))
        assert dd.ddppo_preempt_decide(cfg, 4, s, f) == preempt.should_stop(s, 128, f, 3, 32)
    assert dd.ddppo_preempt_threshold(dd.preempt_cfg(60, 128, min_steps=10), 4) == (3, 10)
    with pytest.raises(dd.DdppoError):
        dd.ddppo_preempt_threshold(dd.preempt_cfg(0, 128), 4)


def test_layout_hash_distinguishes_configs():
    """the rendezvous layout hash must change with the model and with the learner geometry."""
    base = dict(E=4, T=128, ld=132, minibatches=2, epochs=2)
    h = {arch: dd.ddppo_layout_hash(dd.model_desc(arch), **base) for arch in ("toy", "gps", "depth", "rgbd")}
    assert len(set(h.values())) == 4
    assert dd.ddppo_layout_hash(dd.model_desc("gps"), **base) == h["gps"]  # deterministic
    for k, v in (("E", 8), ("T", 64), ("ld", 136), ("minibatches", 4), ("epochs", 1)):
        assert dd.ddppo_layout_hash(dd.model_desc("depth"), **dict(base, **{k: v})) != h["depth"], k


def test_rollout_steps_is_the_a10_input():
    """ddppo_rollout_steps = sum_e min(L_e, T) (P:L635 step accounting; a preempted env counts its
    L_w) -- brute force over random lengths, including L = 0 and L > T; bad input rejected."""
    rng = np.random.default_rng(5)
    for _ in range(200):
        E, T = int(rng.integers(1, 40)), int(rng.integers(1, 300))
        L = rng.integers(0, 2 * T, E).astype(np.int32)
        assert dd.ddppo_rollout_steps(L, T) == sum(min(int(x), T) for x in L)
    with pytest.raises(dd.DdppoError):
        dd.ddppo_rollout_steps(np.array([3, -1], np.int32), 8)
    with pytest.raises(dd.DdppoError):
        dd.ddppo_rollout_steps(np.array([3], np.int32), 0)
