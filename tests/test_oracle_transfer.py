"""Pins for oracle.transfer / the transfer mechanics of oracle.models and oracle.learner (NEXT-4,
P:L401-416)."""
import numpy as np

import synth
from oracle import learner, models, ppo, transfer


def test_splitmix64_published_vector():
    # SplitMix64 with state 0: the first output mixes 0 + golden gamma -> 0xE220A8397B1DCDAF (the
    # published reference sequence of Steele, Lea & Flood's generator)
    assert transfer.splitmix64(transfer.GAMMA) == 0xE220A8397B1DCDAF
    assert transfer.splitmix64(2 * transfer.GAMMA) == 0x6E789E6AA1B965F4


def _entries(arch):
    offs, P = models.offsets(arch)
    fans = {n: f for n, _, f in models.layout(arch)}
    return [(o, int(np.prod(s)), fans[k]) for k, (o, s) in offs.items()], P


def test_reinit_critic_only_value_head():
    ent, P = _entries("depth")
    p0 = synth.init_params(ent, P, 3)
    rng = np.random.default_rng(0)
    m0, v0 = rng.normal(size=P).astype(np.float32), rng.random(P).astype(np.float32)
    p1, m1, v1 = transfer.reinit_critic("depth", p0, m0, v0, seed=7)
    p2, _, _ = transfer.reinit_critic("depth", p0, m0, v0, seed=7)
    p3, _, _ = transfer.reinit_critic("depth", p0, m0, v0, seed=8)
    assert np.array_equal(p1, p2) and not np.array_equal(p1, p3)  # deterministic in the seed
    offs, _ = models.offsets("depth")
    (ow, sw), (ob, _) = offs["head.weight"], offs["head.bias"]
    head = np.zeros(P, bool)
    head[ow + 4 * sw[1]:ow + 5 * sw[1]] = True
    head[ob + 4] = True
    assert np.array_equal(p1[~head], p0[~head]) and np.array_equal(m1[~head], m0[~head])
    assert np.all(m1[head] == 0) and np.all(v1[head] == 0)
    bound = 1.0 / np.sqrt(512)
    vals = p1[head].astype(np.float64)
    assert np.all(np.abs(vals) <= bound) and not np.array_equal(vals, p0[head])
    # U(-b, b): mean 0, variance b^2 / 3 (513 samples: 4-sigma bands)
    n = vals.size
    assert abs(vals.mean()) < 4 * bound / np.sqrt(3 * n)
    assert abs(vals.var() / (bound ** 2 / 3) - 1) < 4 * np.sqrt(0.8 / n)


def _depth_case(T=2, E=2):
    ent, P = _entries("depth")
    p = synth.init_params(ent, P, 5).astype(np.float64)
    ro = synth.rollout(E, T, 9, obs_shape=(1, 64, 64))
    batch = {"goal": ro["goal"].astype(np.float64), "prev_action": ro["prev_action"][:, :T],
             "mask": ro["mask"][:, :T].astype(np.float64), "h0": ro["h0"].astype(np.float64),
             "obs": ro["obs"].astype(np.float64), "c0": ro["c0"].astype(np.float64)}
    lin = {k: v.astype(np.float64) if v.dtype != np.int32 else v for k, v in synth.random_loss_inputs(E * T, 4).items()}
    return p, batch, lin


def _loss(p, batch, lin, extra=None, freeze_encoder=False):
    lg, v, cache = models.forward("depth", p, batch)
    B, T = v.shape
    st, dl, dv = ppo.loss_and_grad(lg.reshape(B * T, -1), v.reshape(-1), lin["actions"], lin["logp_old"],
                                   lin["values_old"], lin["returns"], lin["adv"], np.ones(B * T, bool))
    g = models.backward("depth", p, cache, dl.reshape(B, T, -1), dv.reshape(B, T), extra=extra,
                        freeze_encoder=freeze_encoder)
    return st["total"], g


def test_dgoal_matches_finite_differences():
    """The gradient wrt the goal input (the planner's signal through a frozen controller)."""
    p, batch, lin = _depth_case()
    extra = {}
    _, g = _loss(p, batch, lin, extra)
    dgoal = extra["dgoal"]
    h = 1e-6
    for (b, t, c) in [(0, 0, 0), (1, 1, 2), (0, 1, 1), (1, 0, 0)]:
        bp = {k: v.copy() if isinstance(v, np.ndarray) else v for k, v in batch.items()}
        bm = {k: v.copy() if isinstance(v, np.ndarray) else v for k, v in batch.items()}
        bp["goal"][b, t, c] += h
        bm["goal"][b, t, c] -= h
        fd = (_loss(p, bp, lin)[0] - _loss(p, bm, lin)[0]) / (2 * h)
        assert abs(fd - dgoal[b, t, c]) <= 1e-6 * max(1.0, abs(fd)), (b, t, c, fd, dgoal[b, t, c])


def test_freeze_encoder_gradient_and_update():
    """A frozen encoder gets no gradient (its entries 0) while every other entry equals the unfrozen
    gradient; through the learner step its parameters stay bit-identical and the rest moves."""
    p, batch, lin = _depth_case()
    _, g_full = _loss(p, batch, lin)
    _, g_frz = _loss(p, batch, lin, freeze_encoder=True)
    enc = transfer.encoder_mask("depth", p.size)
    assert np.all(g_frz[enc] == 0) and np.array_equal(g_frz[~enc], g_full[~enc])
    assert np.abs(g_full[enc]).max() > 0
    ent, P = _entries("depth")
    p0 = synth.init_params(ent, P, 6)
    ro = synth.rollout(4, 4, 10, obs_shape=(1, 64, 64))
    pm = synth.perms(10, 0, 1, 4)
    po, mo, vo, _, _ = learner.learner_step("depth", p0, np.zeros(P), np.zeros(P), 0, [ro], [pm],
                                            dict(epochs=1, minibatches=2, freeze_encoder=True))
    assert np.array_equal(po[enc], p0[enc].astype(np.float64)) and np.all(mo[enc] == 0) and np.all(vo[enc] == 0)
    assert np.abs(po[~enc] - p0[~enc]).max() > 1e-4
