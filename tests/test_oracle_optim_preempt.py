"""Pins for oracle.optim (step a8), oracle.preempt (a9) and oracle.minibatch (a4)."""
import json
import os

import numpy as np
import torch

import synth
from oracle import minibatch, optim, preempt

GOLD = json.load(open(os.path.join(os.path.dirname(__file__), "golden", "spec_examples.json")))


def test_allreduce_spec_example():
    g = GOLD["allreduce_N2"]
    assert np.array_equal(optim.allreduce_mean([np.array(x, float) for x in g["inputs"]]), g["mean"])
    x = np.random.default_rng(0).normal(size=11)
    assert np.array_equal(optim.allreduce_mean([x]), x)


def test_adam_first_step_and_zero_grad_and_freeze():
    g = GOLD["adam_first_step"]
    p, m, v, _ = optim.adam_step(np.zeros(1), np.array([g["g"]]), np.zeros(1), np.zeros(1), 1,
                                 lr=g["lr"], max_grad_norm=None)
    assert abs(p[0] - g["delta"]) < 1e-12
    p0 = np.random.default_rng(1).normal(size=7)
    p, m, v, _ = optim.adam_step(p0, np.zeros(7), np.zeros(7), np.zeros(7), 1)
    assert np.array_equal(p, p0)
    fr = np.ones(7, bool)
    p, m, v, _ = optim.adam_step(p0, np.ones(7), np.zeros(7), np.zeros(7), 1, freeze=fr)
    assert np.array_equal(p, p0) and not m.any()


def test_adam_and_clip_match_torch():
    rng = np.random.default_rng(2)
    P = 37
    p0 = rng.normal(size=P)
    tp = torch.tensor(p0.copy(), requires_grad=True)
    opt = torch.optim.Adam([tp], lr=2.5e-4, betas=(0.9, 0.999), eps=1e-8)
    p, m, v = p0.copy(), np.zeros(P), np.zeros(P)
    for step in range(1, 6):
        g = rng.normal(size=P) * (3.0 if step % 2 else 0.01)
        tp.grad = torch.tensor(g.copy())
        torch.nn.utils.clip_grad_norm_([tp], 0.5)
        opt.step()
        p, m, v, _ = optim.adam_step(p, g, m, v, step, max_grad_norm=0.5)
        assert np.max(np.abs(p - tp.detach().numpy())) < 1e-14


def test_preempt_spec_arithmetic():
    g = GOLD["preempt_p60_N4_K"]
    assert preempt.threshold_count(g["p_percent"], g["N"]) == g["K"]
    assert preempt.min_steps(128) == GOLD["preempt_min_T128"]["min_steps"]
    assert not preempt.should_stop(16, 128, 3, 3, 32)
    assert preempt.threshold_count(60, 8) == 5 and preempt.threshold_count(60, 8, other_workers=True) == 5
    assert preempt.threshold_count(60, 2) == 2 and preempt.threshold_count(60, 2, other_workers=True) == 1
    assert preempt.threshold_count(60, 1, other_workers=True) == 1


def test_closed_form_equals_tick_simulation():
    rng = np.random.default_rng(3)
    for trial in range(1500):
        N = int(rng.choice([1, 2, 3, 4, 5, 8]))
        T = int(rng.integers(4, 65))
        p = int(rng.choice([10, 50, 60, 80, 100]))
        costs = rng.integers(1, int(rng.integers(2, 30)), (N, T))
        ow = bool(trial % 5 == 0)
        L1 = preempt.closed_form_lengths(costs, T, p, other_workers=ow)
        L2, ticks, polls = preempt.simulate_ticks(costs, T, p, other_workers=ow)
        assert np.array_equal(L1, L2), (costs, T, p)
        ms = preempt.min_steps(T)
        K = preempt.threshold_count(p, N, ow)
        assert L1.min() >= min(ms, T)  # safety
        assert (L1 == T).sum() >= K  # at least K natural finishers
        fins = [f for _, f, _ in polls]
        assert all(a <= b for a, b in zip(fins, fins[1:])) and fins[-1] <= N  # monotone
        if p == 100 and not ow:
            assert np.all(L1 == T)


def test_straggler_bounds_and_accounting():
    costs = synth.straggler_costs(0, 8, 128)
    costs[3] *= 10  # one 10x-slow worker
    L = preempt.closed_form_lengths(costs, 128, 60)
    assert 32 <= L[3] < 128
    col, pre = preempt.step_accounting(L, 16, 128)
    assert col + pre == 8 * 16 * 128 and col == int(16 * L.sum())


def test_minibatch_exact_cover():
    pm = synth.perms(0, 0, 2, 4)
    length = np.array([128, 32, 128, 77])
    for e in range(2):
        seen = []
        for j in range(2):
            envs = minibatch.minibatch_envs(pm[e], 2, j)
            assert len(envs) == 2
            seen += minibatch.samples(envs, length)
        assert sorted(seen) == sorted((n, t) for n in range(4) for t in range(length[n]))
    assert len(minibatch.samples(pm[0], [128, 32, 128, 77])) == 365
