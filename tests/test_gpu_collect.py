"""NEXT-1, the collection side, on the GPU:
  * ddppo_policy_act (batched single-step inference) against the oracle's forward of that step:
    logits / values / the new recurrent state; the sampled actions against oracle.sample on the
    kernels' logits (bit-exact but for draws within rounding of a cumulative boundary); logp 1e-5;
  * a collect + learn cycle through paper_1911_00357_b200.collect: the rollout is self-consistent
    (mask / previous-action semantics; logp_old is what the training forward assigns to the collected
    actions, so the first minibatch runs at ratio ~ 1: PPO's common case); lengths under the
    preemption protocol in wall-clock ticks equal the closed form (N = 1 here; N = 2 in
    test_gpu_multi.py)."""
import numpy as np
import pytest
import torch

import paper_1911_00357_b200 as dd
import synth
from oracle import models, preempt, sample
from paper_1911_00357_b200.collect import Collector, run_cycles
from paper_1911_00357_b200.learner import Learner

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def ctx():
    c = dd.Context(0, 1, device=0)
    yield c
    c.close()


def rel_l2(a, b):
    return float(np.linalg.norm(np.asarray(a, np.float64) - b) / max(np.linalg.norm(b), 1e-30))


def _params(arch, seed, hidden=None):
    desc = dd.model_desc(arch, hidden)
    lay = dd.param_layout(desc)
    P = dd.param_count(desc)
    return desc, synth.init_params([(off, int(np.prod(s)), fan) for _, off, s, fan in lay], P, seed)


@pytest.mark.parametrize("arch,E,hidden", [("gps", 4, None), ("gps", 13, None), ("depth", 4, None), ("depth", 12, None),
                                           ("rgbd", 3, None), ("depth", 5, 1024)])  # NEXT-3's 1024-d LSTM
def test_policy_act_matches_oracle_step(ctx, arch, E, hidden):
    desc, p0 = _params(arch, 2, hidden)
    H = desc.hidden
    layers = 2 if arch == "rgbd" else 1
    vis = arch != "gps"
    rng = np.random.default_rng(E)
    env = synth.PointGoalEnv(E, 5, obs=None if arch == "gps" else arch, H=256 if arch == "rgbd" else 64)
    for _ in range(3):  # mid-episode states (some envs just reset)
        env.step(rng.integers(0, 4, E))
    g, pa, m, frames = env.observe()
    h0 = rng.normal(0, 0.1, (E, layers * H)).astype(np.float32)
    c0 = rng.normal(0, 0.1, (E, layers * H)).astype(np.float32)
    cu = lambda a: torch.from_numpy(np.ascontiguousarray(a)).cuda()  # noqa: E731
    prev = np.zeros((E, 2), np.int32)
    prev[:, 0] = pa
    mask = np.zeros((E, 2), np.float32)
    mask[:, 0] = m
    obs = {k: t.cuda() for k, t in dd.visual_obs(frames[:, None], arch == "rgbd").items()} if vis else {}
    h_out, c_out = torch.zeros((E, layers * H), device="cuda"), torch.zeros((E, layers * H), device="cuda")
    ab = dd.make_act_batch(cu(g.reshape(E, 1, 3)), cu(prev), cu(mask), cu(h0), h_out, E, 1, 2, 0, 17, 3,
                           obs=obs.get("obs"), obs_rgb=obs.get("obs_rgb"), c_in=cu(c0) if vis else None,
                           c_out=c_out if vis else None)
    acts, logp, vals = (torch.zeros(E, dtype=torch.int32, device="cuda"), torch.zeros(E, device="cuda"),
                        torch.zeros(E, device="cuda"))
    lg = torch.zeros((E, 4), device="cuda")
    ws = torch.empty(dd.act_workspace_size(desc, E) // 4 + 64, device="cuda")
    dd.ddppo_policy_act(ctx, desc, cu(p0), ab, acts, logp, vals, ws, logits=lg)
    torch.cuda.synchronize()
    ctx.check()
    batch = {"goal": g.reshape(E, 1, 3).astype(np.float64), "prev_action": pa.reshape(E, 1),
             "mask": m.reshape(E, 1).astype(np.float64), "h0": h0.astype(np.float64)}
    if vis:
        batch.update(obs=frames[:, None].astype(np.float64), c0=c0.astype(np.float64))
    lo, vo, cache = models.forward(arch, p0, batch, hidden=H)
    lim = 1e-3 if vis else 2e-2
    assert rel_l2(lg.cpu().numpy(), lo[:, 0]) < lim and rel_l2(vals.cpu().numpy(), vo[:, 0]) < lim
    ho, co = h_out.cpu().numpy(), c_out.cpu().numpy()
    if arch == "rgbd":
        h_ref = [cache["rnn"][1]["x"][:, 0], cache["h"][:, 0]]
        c_ref = [cache["rnn"][0]["c"][:, 0], cache["rnn"][1]["c"][:, 0]]
    else:
        h_ref = [cache["h"][:, 0]]
        c_ref = [cache["rnn"]["c"][:, 0]] if vis else []
    for l, ref in enumerate(h_ref):
        assert rel_l2(ho[:, l * H:(l + 1) * H], ref) < lim, ("h", l)
    for l, ref in enumerate(c_ref):
        assert rel_l2(co[:, l * H:(l + 1) * H], ref) < lim, ("c", l)
    # the draw: oracle.sample on the kernels' own logits (the decision is the kernels' fp32 one)
    a_o, lp_o, margin = sample.sample(lg.cpu().numpy(), 17, 3)
    a_g = acts.cpu().numpy()
    diff = a_g != a_o
    assert np.all(margin[diff] < 1e-6), (a_g, a_o, margin)
    same = ~diff
    assert np.allclose(logp.cpu().numpy()[same], lp_o[same], atol=1e-5)
    # greedy
    ab.greedy = 1
    dd.ddppo_policy_act(ctx, desc, cu(p0), ab, acts, logp, vals, ws, logits=lg)
    torch.cuda.synchronize()
    assert np.array_equal(acts.cpu().numpy(), np.argmax(lg.cpu().numpy(), axis=1))


def test_collect_learn_cycle_depth(ctx):
    c = synth.CONFIGS["depth"]
    E, T = c["E"], 24
    desc, p0 = _params("depth", 4)
    lrn = Learner(ctx, "depth", E, T, c["epochs"], c["minibatches"], params=p0, normalize_adv=True)
    env = synth.PointGoalEnv(E, 9, obs="depth")
    col = Collector(lrn, env, seed=9)
    ro = col.collect(T)
    # rollout semantics: mask_t = 1 - done_{t-1}; prev_action_t = action_{t-1} (start token after a reset)
    for t in range(1, T):
        assert np.array_equal(ro["mask"][:, t], 1.0 - ro["done"][:, t - 1])
        exp_prev = np.where(ro["done"][:, t - 1] == 1, synth.START_TOKEN, ro["action"][:, t - 1])
        assert np.array_equal(ro["prev_action"][:, t], exp_prev)
    # logp_old / V are the policy's own: the training forward over the whole rollout reproduces them
    # (recurrent state carried across steps inside one launch vs step by step through act)
    cu = lambda a: torch.from_numpy(np.ascontiguousarray(a)).cuda()  # noqa: E731
    vo = {k: t.cuda() for k, t in dd.visual_obs(ro["obs"], False).items()}
    env_idx = np.arange(E, dtype=np.int32)
    batch = dd.make_batch(cu(ro["goal"]), cu(ro["prev_action"]), cu(ro["mask"]), cu(ro["h0"]),
                          cu(ro["length"]), cu(env_idx[:2]), E, T, ro["ld"], 2, T, 2 * T, obs=vo["obs"],
                          c0=cu(ro["c0"]))
    ws = torch.zeros(dd.workspace_size(desc, 2, T) // 4 + 64, device="cuda")
    lg, vl = torch.zeros((2, T, 4), device="cuda"), torch.zeros((2, T), device="cuda")
    dd.ddppo_policy_fwd(ctx, desc, lrn.params, batch, lg, vl, ws)
    torch.cuda.synchronize()
    z = lg.cpu().numpy().astype(np.float64)
    lp = z - np.log(np.exp(z - z.max(-1, keepdims=True)).sum(-1, keepdims=True)) - z.max(-1, keepdims=True)
    lp_a = np.take_along_axis(lp, ro["action"][:2, :T, None].astype(np.int64), -1)[..., 0]
    assert np.max(np.abs(lp_a - ro["logp_old"][:2, :T])) < 2e-3
    assert np.max(np.abs(vl.cpu().numpy() - ro["val"][:2, :T])) < 2e-3 * max(1.0, np.abs(ro["val"]).max())
    # the learner step on it: the first minibatch runs at ratio ~ 1 (approx-KL ~ 0, nothing clipped)
    lrn.load_rollout(ro, synth.perms(9, 0, c["epochs"], E))
    st = lrn.step().cpu().numpy()
    ctx.check()
    assert abs(st[0, 4]) < 1e-3 and st[0, 3] == 0.0  # approx_kl, clip_frac of minibatch 0
    # two more P:L628 cycles, and the preemption protocol in wall-clock ticks (N = 1: nobody waits)
    sps, log = run_cycles(lrn, col, T, lambda i: synth.perms(9, i + 1, c["epochs"], E), cycles=2, timed=1)
    assert sps > 0 and all(L == T for L, *_ in log)
    costs = synth.straggler_costs(3, 1, T)[0]
    ro2 = col.collect(T, costs=costs, p_percent=60, tick_s=1e-4)
    assert int(ro2["length"][0]) == preempt.closed_form_lengths(costs[None], T, 60)[0] == T
