"""NEXT-4 transfer mechanics on the GPU: critic re-initialisation (bit-exact against the
oracle's counter-based generator), a per-entry freeze mask inside ddppo_learner_step, and the goal-
input gradient of the differentiable neural controller.  The frozen visual encoder inside the
learner step is pinned by test_gpu_parity.py::test_learner_chain_parity (frozen cases)."""
import numpy as np
import pytest
import torch

import paper_1911_00357_b200 as dd
import synth
from oracle import learner, models, transfer
from paper_1911_00357_b200.learner import Learner, reinit_critic

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def ctx():
    c = dd.Context(0, 1, device=0)
    yield c
    c.close()


def _p0(arch, seed):
    desc = dd.model_desc(arch)
    lay = dd.param_layout(desc)
    P = dd.param_count(desc)
    return desc, lay, P, synth.init_params([(off, int(np.prod(s)), fan) for _, off, s, fan in lay], P, seed)


def rel_l2(a, b):
    return float(np.linalg.norm(np.asarray(a, np.float64) - b) / max(np.linalg.norm(b), 1e-30))


@pytest.mark.parametrize("arch", ["toy", "gps", "depth", "rgbd"])
def test_reinit_critic_bit_exact(ctx, arch):
    desc, lay, P, p0 = _p0(arch, 1)
    rng = np.random.default_rng(2)
    m0, v0 = rng.normal(size=P).astype(np.float32), rng.random(P).astype(np.float32)
    p, m, v = (torch.from_numpy(x.copy()).cuda() for x in (p0, m0, v0))
    dd.ddppo_reinit_critic(ctx, desc, p, m, v, 1234)
    torch.cuda.synchronize()
    po, mo, vo = transfer.reinit_critic(arch, p0, m0, v0, 1234, hidden=desc.hidden)
    assert np.array_equal(p.cpu().numpy(), po) and np.array_equal(m.cpu().numpy(), mo)
    assert np.array_equal(v.cpu().numpy(), vo)
    assert not np.array_equal(po, p0)


# the frozen-encoder learner step itself: tests/test_gpu_parity.py::test_learner_chain_parity[...-True]


def test_freeze_mask_learner_step(ctx):
    c = synth.CONFIGS["gps"]
    desc, lay, P, p0 = _p0("gps", 5)
    mask = (np.random.default_rng(6).random(P) < 0.25).astype(np.uint8)
    lrn = Learner(ctx, "gps", c["E"], 32, 2, 2, params=p0, normalize_adv=True, freeze_mask=mask)
    lrn.load_rollout(synth.rollout(c["E"], 32, 7), synth.perms(7, 0, 2, c["E"]))
    lrn.step()
    torch.cuda.synchronize()
    ctx.check()
    got = lrn.params.cpu().numpy()
    f = mask.astype(bool)
    assert np.array_equal(got[f], p0[f]) and np.abs(got[~f] - p0[~f]).max() > 1e-4


def test_controller_goal_gradient(ctx):
    """dL/d(goal input) of the Depth agent (the signal a planner receives through the frozen
    controller) against the oracle with the kernels' decisions adopted: 2e-2."""
    from tests.test_gpu_parity import _adopt_decisions
    desc, lay, P, params = _p0("depth", 8)
    E, T, B = 2, 6, 2
    ro = synth.rollout(E, T, 9, obs_shape=(1, 64, 64))
    env_idx = np.array([1, 0], np.int32)
    cu = lambda a: torch.from_numpy(np.ascontiguousarray(a)).cuda()  # noqa: E731
    vo_ = {k: t.cuda() for k, t in dd.visual_obs(ro["obs"], False).items()}
    dgoal = torch.zeros((B * T, 3), device="cuda")
    batch = dd.make_batch(cu(ro["goal"]), cu(ro["prev_action"]), cu(ro["mask"]), cu(ro["h0"]), cu(ro["length"]),
                          cu(env_idx), E, T, ro["ld"], B, T, B * T, obs=vo_["obs"], c0=cu(ro["c0"]), dgoal=dgoal,
                          freeze_encoder=True)
    ws = torch.zeros(dd.workspace_size(desc, B, T) // 4 + 64, device="cuda")
    lg, vl = torch.zeros((B, T, 4), device="cuda"), torch.zeros((B, T), device="cuda")
    pg = cu(params)
    dd.ddppo_policy_fwd(ctx, desc, pg, batch, lg, vl, ws)
    dec = dd.ddppo_debug_depth_decisions(ctx, desc, batch, ws).cpu().numpy()
    rng = np.random.default_rng(10)
    dl = rng.normal(0, 1e-2, (B, T, 4)).astype(np.float32)
    dv = rng.normal(0, 1e-2, (B, T)).astype(np.float32)
    grad = torch.full((P,), 3.0, device="cuda")
    dd.ddppo_policy_bwd(ctx, desc, pg, batch, cu(dl), cu(dv), grad, ws)
    torch.cuda.synchronize()
    ctx.check()
    ob = {"goal": ro["goal"][env_idx], "prev_action": ro["prev_action"][env_idx, :T], "mask": ro["mask"][env_idx, :T],
          "h0": ro["h0"][env_idx], "obs": ro["obs"][env_idx], "c0": ro["c0"][env_idx]}
    _, _, cache = models.forward("depth", params, ob)
    _adopt_decisions("depth", params, ob, cache, dec, B * T)
    extra = {}
    go = models.backward("depth", params, cache, dl.astype(np.float64), dv.astype(np.float64), extra=extra,
                         freeze_encoder=True)
    assert rel_l2(dgoal.cpu().numpy(), extra["dgoal"].reshape(B * T, 3)) < 2e-2
    g = grad.cpu().numpy()
    enc = transfer.encoder_mask("depth", P)
    assert np.all(g[enc] == 0)  # frozen encoder: no gradient
    assert rel_l2(g[~enc], go[~enc]) < 2e-2
