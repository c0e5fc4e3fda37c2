"""Pins for oracle.gae / oracle.advnorm (steps a2, a3) -- closed forms, brute force, invariants."""
import json
import os

import numpy as np
import pytest

from oracle import advnorm, gae

GOLD = json.load(open(os.path.join(os.path.dirname(__file__), "golden", "spec_examples.json")))


def _rand_buf(rng, E, T, p_done=0.1):
    rew = rng.normal(size=(E, T + 1))
    val = rng.normal(size=(E, T + 1))
    done = (rng.random((E, T + 1)) < p_done).astype(np.uint8)
    length = rng.integers(1, T + 1, E)
    return rew, val, done, length


def test_single_terminal_step():
    g = GOLD["gae_single_terminal"]
    for gamma in (0.0, 0.5, 0.99, 1.0):
        for tau in (0.0, 0.95, 1.0):
            a, r = gae.gae([[g["r"], 0]], [[g["v0"], 7.0]], [[g["done"], 0]], [1], gamma, tau)
            assert a[0, 0] == g["adv"] and r[0, 0] == g["ret"]


def test_tau1_closed_form_discounted_return_minus_value():
    """tau=1: A_t = sum_{k=t}^{e} g^{k-t} r_k + g^{e+1-t} v_{e+1} [no done in t..e] - v_t (P:L127 MC form)."""
    rng = np.random.default_rng(0)
    for trial in range(300):
        E, T = 3, int(rng.integers(1, 20))
        rew, val, done, length = _rand_buf(rng, E, T)
        gamma = float(rng.choice([0.0, 0.5, 0.99, 1.0]))
        a, _ = gae.gae(rew, val, done, length, gamma, 1.0)
        for n in range(E):
            L = length[n]
            for t in range(L):
                tot, disc, boot = 0.0, 1.0, True
                for k in range(t, L):
                    tot += disc * rew[n, k]
                    if done[n, k]:
                        boot = False
                        break
                    disc *= gamma
                if boot:
                    tot += disc * val[n, L]
                assert abs(a[n, t] - (tot - val[n, t])) < 1e-9 * (1 + abs(tot))


def test_tau0_is_td_error():
    rng = np.random.default_rng(1)
    rew, val, done, length = _rand_buf(rng, 5, 33)
    a, _ = gae.gae(rew, val, done, length, 0.99, 0.0)
    for n in range(5):
        for t in range(length[n]):
            td = rew[n, t] + 0.99 * val[n, t + 1] * (1 - done[n, t]) - val[n, t]
            assert abs(a[n, t] - td) < 1e-12


def test_brute_force_quadratic():
    """A_t = sum_l (g tau)^l prod_{j<l}(1-d_{t+j}) delta_{t+l}."""
    rng = np.random.default_rng(2)
    for _ in range(100):
        E, T = 2, int(rng.integers(1, 25))
        rew, val, done, length = _rand_buf(rng, E, T, 0.2)
        gamma, tau = 0.99, 0.95
        a, r = gae.gae(rew, val, done, length, gamma, tau)
        for n in range(E):
            L = length[n]
            delta = [rew[n, k] + gamma * val[n, k + 1] * (1 - done[n, k]) - val[n, k] for k in range(L)]
            for t in range(L):
                s, w = 0.0, 1.0
                for l in range(L - t):
                    s += w * delta[t + l]
                    w *= gamma * tau * (1 - done[n, t + l])
                assert abs(a[n, t] - s) < 1e-10
                assert abs(r[n, t] - (a[n, t] + val[n, t])) < 1e-12  # R = A + V
            assert np.all(a[n, L:] == 0)


def test_discounted_return_when_value_zero():
    """tau=1, V=0, no truncation bootstrap => A equals the discounted return of Eq.1."""
    rng = np.random.default_rng(3)
    T = 17
    rew = rng.normal(size=(1, T + 1))
    val = np.zeros((1, T + 1))
    done = np.zeros((1, T + 1), np.uint8)
    a, _ = gae.gae(rew, val, done, [T], 0.9, 1.0)
    for t in range(T):
        assert abs(a[0, t] - sum(0.9 ** (k - t) * rew[0, k] for k in range(t, T))) < 1e-12


def test_adv_norm_moments_and_rank_concat():
    rng = np.random.default_rng(4)
    advs, lens = [], []
    for r in range(3):
        E, T = 4, 16
        rew, val, done, length = _rand_buf(rng, E, T)
        a, _ = gae.gae(rew, val, done, length, 0.99, 0.95)
        advs.append(a)
        lens.append(length)
    st = advnorm.combine([gae.adv_stats(a, l) for a, l in zip(advs, lens)])
    cat = np.concatenate([a[np.arange(a.shape[1])[None] < l[:, None]] for a, l in zip(advs, lens)])
    assert st[2] == cat.size
    assert abs(st[0] - cat.sum()) < 1e-9 and abs(st[1] - (cat ** 2).sum()) < 1e-9
    mu, inv = advnorm.mean_invstd(st, 1e-5)
    z = advnorm.normalize(cat, mu, inv)
    sigma = cat.std(ddof=1)
    assert abs(z.mean()) < 1e-12
    assert abs(z.std(ddof=1) - sigma / (sigma + 1e-5)) < 1e-12


def test_adv_norm_identity_flag_off():
    from oracle import ppo
    import synth
    x = synth.random_loss_inputs(16, 0)
    valid = np.ones(16, bool)
    s1, d1, v1 = ppo.loss_and_grad(x["logits"], x["values"], x["actions"], x["logp_old"], x["values_old"],
                                   x["returns"], x["adv"], valid, mean_invstd=None)
    s2, d2, v2 = ppo.loss_and_grad(x["logits"], x["values"], x["actions"], x["logp_old"], x["values_old"],
                                   x["returns"], x["adv"], valid, mean_invstd=(0.0, 1.0))
    assert np.array_equal(d1, d2) and s1["total"] == s2["total"]


@pytest.mark.parametrize("gamma,tau", [(0.99, 0.95)])
def test_paper_hparams(gamma, tau):
    h = GOLD["hparams"]
    assert (h["gamma"], h["tau"]) == (gamma, tau)
