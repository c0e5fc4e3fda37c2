"""GPU parity of every step of the hot path against the oracle, through the C ABI (-m gpu).

Tolerances (BASELINE.json north_star):
  GAE / normalisation  |g-o| <= 1e-5|o| + 1e-5 max|o| (per env row)          (fp32 path)
  loss / dlogits / Adam |g-o| <= 1e-4|o| + 1e-4 max|o| (per tensor)           (fp32 path)
  toy network           same 1e-4 form
  GPS network (fp16/bf16 tensor-core recurrence) per-tensor relative L2 <= 2e-2
  integers (lengths, counts, preemption) bit-exact
"""
import numpy as np
import pytest
import torch

import synth
from oracle import advnorm, convnets, gae, learner, minibatch, models, optim, ppo

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def dd():
    if not torch.cuda.is_available():
        pytest.skip("needs a GPU")
    import paper_1911_00357_b200 as m
    return m


@pytest.fixture(scope="module")
def ctx(dd):
    c = dd.Context(0, 1, device=0)
    yield c
    c.close()


def cu(a, dtype=None):
    t = torch.from_numpy(np.ascontiguousarray(a))
    if dtype is not None:
        t = t.to(dtype)
    return t.cuda()


def close_rel(g, o, rel, name=""):
    g = np.asarray(g, dtype=np.float64)
    o = np.asarray(o, dtype=np.float64)
    scale = np.max(np.abs(o)) if o.size else 0.0
    bad = np.abs(g - o) > rel * np.abs(o) + rel * scale + 1e-30
    assert not bad.any(), f"{name}: {bad.sum()} / {bad.size} mismatches, max err {np.max(np.abs(g - o))}, scale {scale}"


def close_update(p_new, p_old, p_ref, rel, name=""):
    """fp32 parameters after an update vs the fp64 oracle's: the update within `rel` (elementwise,
    with the tensor-scale floor of close_rel) plus half an fp32 ulp of the parameter -- the master
    weights are fp32 (Z24), so theta + delta is rounded to the fp32 grid around theta (GN gamma = 1
    gives ulp 1.2e-7 against |delta| ~ lr = 2.5e-4)."""
    p_new, p_old, p_ref = (np.asarray(a, dtype=np.float64) for a in (p_new, p_old, p_ref))
    d, d_ref = p_new - p_old, p_ref - p_old
    half_ulp = np.spacing(np.abs(p_ref).astype(np.float32)).astype(np.float64)
    bad = np.abs(d - d_ref) > rel * np.abs(d_ref) + rel * np.abs(d_ref).max() + half_ulp
    assert not bad.any(), f"{name}: {bad.sum()} / {bad.size} mismatches, max err {np.max(np.abs(d - d_ref))}"


def rel_l2(g, o):
    g = np.asarray(g, dtype=np.float64)
    o = np.asarray(o, dtype=np.float64)
    return np.linalg.norm(g - o) / max(np.linalg.norm(o), 1e-30)


# ------------------------------------------------------------------ a2 GAE + a3 stats
def _gae_case(dd, ctx, E, T, seed, lengths=None, gamma=0.99, tau=0.95, p_done=0.05, ld=None, done_mode=None):
    rng = np.random.default_rng(seed)
    ld = ld or synth.ld_for(T)
    rew = rng.normal(size=(E, ld)).astype(np.float32)
    val = rng.normal(size=(E, ld)).astype(np.float32)
    done = (rng.random((E, ld)) < p_done).astype(np.uint8)
    if done_mode == "all":
        done[:] = 1
    elif done_mode == "none":
        done[:] = 0
    length = np.full(E, T, np.int32) if lengths is None else np.asarray(lengths, np.int32)
    if done_mode == "last":
        done[:] = 0
        done[np.arange(E), length - 1] = 1
    adv = torch.full((E, ld), 7.0, device="cuda")
    ret = torch.full((E, ld), 7.0, device="cuda")
    st = torch.zeros(3, dtype=torch.float64, device="cuda")
    dd.ddppo_gae(ctx, cu(rew), cu(val), cu(done), cu(length), E, T, ld, gamma, tau, adv, ret, st)
    torch.cuda.synchronize()
    a_o, r_o = gae.gae(rew, val, done, length, gamma, tau)
    A = adv.cpu().numpy()[:, :T]
    R = ret.cpu().numpy()[:, :T]
    Tm = a_o.shape[1]
    for n in range(E):
        close_rel(A[n, :Tm], a_o[n], 1e-5, f"adv row {n}")
        close_rel(R[n, :Tm], r_o[n], 1e-5, f"ret row {n}")
        assert np.all(A[n, length[n]:] == 0) and np.all(R[n, length[n]:] == 0)
    so = gae.adv_stats(a_o, length)
    s = st.cpu().numpy()
    assert s[2] == so[2]
    close_rel(s[:2], so[:2], 1e-5, "stats")
    return s


@pytest.mark.parametrize("E,T", [(2, 4), (4, 128), (16, 128), (37, 200), (5, 7), (3, 1), (300, 64)])
def test_gae_shapes(dd, ctx, E, T):
    rng = np.random.default_rng(E * 1000 + T)
    _gae_case(dd, ctx, E, T, 1)
    _gae_case(dd, ctx, E, T, 2, lengths=rng.integers(1, T + 1, E))


@pytest.mark.parametrize("gamma,tau", [(0.0, 0.95), (1.0, 1.0), (0.99, 0.0), (0.5, 0.5)])
def test_gae_gamma_tau_edges(dd, ctx, gamma, tau):
    _gae_case(dd, ctx, 8, 128, 3, gamma=gamma, tau=tau, lengths=[128, 1, 32, 127, 64, 100, 128, 2])


@pytest.mark.parametrize("mode", ["all", "none", "last"])
def test_gae_done_edges(dd, ctx, mode):
    _gae_case(dd, ctx, 6, 128, 4, lengths=[128, 32, 33, 1, 127, 96], done_mode=mode)


def test_gae_odd_ld_scalar_path(dd, ctx):
    _gae_case(dd, ctx, 9, 128, 5, ld=131, lengths=[128, 5, 64, 1, 100, 128, 77, 31, 32])


def test_gae_empty(dd, ctx):
    st = torch.ones(3, dtype=torch.float64, device="cuda")
    dummy = torch.zeros(8, device="cuda")
    dd.ddppo_gae(ctx, dummy, dummy, torch.zeros(8, dtype=torch.uint8, device="cuda"),
                 torch.zeros(1, dtype=torch.int32, device="cuda"), 0, 4, 8, 0.99, 0.95, dummy, dummy, st)
    torch.cuda.synchronize()
    assert st.cpu().tolist() == [0, 0, 0]


def test_gae_large_sampled(dd, ctx):
    """Microbench-sized buffer (2^16 x 128): sampled env rows against the oracle."""
    E, T = 1 << 16, 128
    ld = synth.ld_for(T)
    rng = np.random.default_rng(6)
    rew = rng.normal(size=(E, ld)).astype(np.float32)
    val = rng.normal(size=(E, ld)).astype(np.float32)
    done = (rng.random((E, ld)) < 0.02).astype(np.uint8)
    length = rng.integers(32, T + 1, E).astype(np.int32)
    adv = torch.empty((E, ld), device="cuda")
    ret = torch.empty((E, ld), device="cuda")
    st = torch.zeros(3, dtype=torch.float64, device="cuda")
    dd.ddppo_gae(ctx, cu(rew), cu(val), cu(done), cu(length), E, T, ld, 0.99, 0.95, adv, ret, st)
    torch.cuda.synchronize()
    idx = rng.choice(E, 64, replace=False)
    a_o, r_o = gae.gae(rew[idx], val[idx], done[idx], length[idx], 0.99, 0.95)
    A = adv.cpu().numpy()[idx]
    for i in range(len(idx)):
        close_rel(A[i, :a_o.shape[1]][:length[idx[i]]], a_o[i][:length[idx[i]]], 1e-5, "adv")
    # the global stats: exact count, sums within fp32-rounding of the full oracle
    a_full, _ = gae.gae(rew, val, done, length, 0.99, 0.95)
    so = gae.adv_stats(a_full, length)
    s = st.cpu().numpy()
    assert s[2] == so[2] == length.sum()
    close_rel(s[:2], so[:2], 1e-5, "stats")


def test_adv_norm(dd, ctx):
    s = _gae_case(dd, ctx, 16, 128, 7, lengths=np.r_[np.full(8, 128), np.full(8, 40)])
    st = torch.tensor(s, dtype=torch.float64, device="cuda")
    mi = torch.zeros(2, device="cuda")
    dd.ddppo_adv_norm(ctx, st, 1e-5, mi)
    torch.cuda.synchronize()
    mu, inv = advnorm.mean_invstd(s, 1e-5)
    close_rel(mi.cpu().numpy(), [mu, inv], 1e-5, "mean_invstd")


# ------------------------------------------------------------------ a6 loss
def _loss_setup(E, T, B, seed, lengths=None):
    rng = np.random.default_rng(seed)
    ro = synth.rollout(E, T, seed, length=lengths, hidden=8)
    a_o, r_o = gae.gae(ro["rew"], ro["val"], ro["done"], ro["length"], 0.99, 0.95)
    ld = ro["ld"]
    adv = np.zeros((E, ld), np.float32)
    ret = np.zeros((E, ld), np.float32)
    adv[:, :a_o.shape[1]] = a_o
    ret[:, :r_o.shape[1]] = r_o
    env_idx = rng.permutation(E)[:B].astype(np.int32)
    L = ro["length"][env_idx]
    T_run = int(L.max())
    logits = rng.normal(0, 1.0, (B, T_run, 4)).astype(np.float32)
    values = (ro["val"][env_idx, :T_run] + rng.normal(0, 0.3, (B, T_run))).astype(np.float32)
    return ro, adv, ret, env_idx, T_run, int(L.sum()), logits, values


@pytest.mark.parametrize("E,T,B,vclip,norm", [(4, 128, 2, True, True), (16, 128, 8, False, True),
                                              (2, 4, 2, True, False), (64, 100, 64, True, True)])
def test_loss_parity(dd, ctx, E, T, B, vclip, norm):
    lengths = np.random.default_rng(E).integers(max(1, T // 4), T + 1, E)
    ro, adv, ret, env_idx, T_run, n_valid, logits, values = _loss_setup(E, T, B, E + T, lengths)
    mis = (0.3, 1.7) if norm else None
    batch = dd.make_batch(cu(ro["goal"]), cu(ro["prev_action"]), cu(ro["mask"]), cu(ro["h0"]), cu(ro["length"]),
                          cu(env_idx), E, T, ro["ld"], B, T_run, n_valid)
    dl = torch.zeros((B, T_run, 4), device="cuda")
    dv = torch.zeros((B, T_run), device="cuda")
    stats = torch.zeros(8, device="cuda")
    keep = [batch]
    dd.ddppo_ppo_loss_grad(ctx, cu(logits), cu(values), batch, cu(ro["action"]), cu(ro["logp_old"]), cu(ro["val"]),
                           cu(ret), cu(adv), cu(np.array(mis, np.float32)) if norm else None,
                           dd.loss_cfg(use_value_clip=vclip, normalize_adv=norm), dl, dv, stats)
    torch.cuda.synchronize()
    ctx.check()
    valid = (np.arange(T_run)[None] < ro["length"][env_idx][:, None]).reshape(-1)
    f = lambda a: a[env_idx, :T_run].reshape(-1)  # noqa: E731
    st, dlo, dvo = ppo.loss_and_grad(logits.reshape(-1, 4), values.reshape(-1), f(ro["action"]), f(ro["logp_old"]),
                                     f(ro["val"]), f(ret), f(adv), valid, use_value_clip=vclip, mean_invstd=mis)
    close_rel(dl.cpu().numpy().reshape(-1, 4), dlo, 1e-4, "dlogits")
    close_rel(dv.cpu().numpy().reshape(-1), dvo, 1e-4, "dvalues")
    s = stats.cpu().numpy()
    for i, k in enumerate(ppo.STAT_NAMES):
        assert abs(s[i] - st[k]) <= 1e-4 * abs(st[k]) + 1e-5, (k, s[i], st[k])
    assert s[6] == n_valid
    del keep


def test_loss_large_sampled(dd, ctx):
    """M = 2^20 samples (B = 8192 envs x 128): sampled rows against the oracle."""
    E, T = 8192, 128
    ld = synth.ld_for(T)
    rng = np.random.default_rng(9)
    M = E * T
    x = synth.random_loss_inputs(M, 10)
    env_idx = np.arange(E, dtype=np.int32)
    length = np.full(E, T, np.int32)
    rowify = lambda a, dt=np.float32: np.pad(a.reshape(E, T), ((0, 0), (0, ld - T))).astype(dt)  # noqa: E731
    batch = dd.make_batch(cu(np.zeros((E, T, 3), np.float32)), None, None, None, cu(length), cu(env_idx), E, T, ld, E,
                          T, M)
    dl = torch.zeros((M, 4), device="cuda")
    dv = torch.zeros(M, device="cuda")
    stats = torch.zeros(8, device="cuda")
    dd.ddppo_ppo_loss_grad(ctx, cu(x["logits"]), cu(x["values"]), batch, cu(rowify(x["actions"], np.int32)),
                           cu(rowify(x["logp_old"])), cu(rowify(x["values_old"])), cu(rowify(x["returns"])),
                           cu(rowify(x["adv"])), None, dd.loss_cfg(normalize_adv=False), dl, dv, stats)
    torch.cuda.synchronize()
    st, dlo, dvo = ppo.loss_and_grad(x["logits"], x["values"], x["actions"], x["logp_old"], x["values_old"],
                                     x["returns"], x["adv"], np.ones(M, bool), use_value_clip=True)
    idx = rng.choice(M, 4096, replace=False)
    close_rel(dl.cpu().numpy()[idx], dlo[idx], 1e-4, "dlogits")
    close_rel(dv.cpu().numpy()[idx], dvo[idx], 1e-4, "dvalues")
    s = stats.cpu().numpy()
    for i, k in enumerate(ppo.STAT_NAMES):
        assert abs(s[i] - st[k]) <= 1e-4 * abs(st[k]) + 1e-5, (k, s[i], st[k])


# ------------------------------------------------------------------ a8 clip + Adam (N = 1)
@pytest.mark.parametrize("P,clip,freeze", [(1001, 0.5, False), (890661, 0.5, True), (7, 0.0, False)])
def test_clip_adam(dd, ctx, P, clip, freeze):
    rng = np.random.default_rng(P)
    p = rng.normal(size=P).astype(np.float32)
    m = rng.normal(0, 0.01, P).astype(np.float32)
    v = rng.uniform(0, 1e-3, P).astype(np.float32)
    fr = (rng.random(P) < 0.3).astype(np.uint8) if freeze else None
    pg, mg, vg = cu(p), cu(m), cu(v)
    po, mo, vo = p.astype(np.float64), m.astype(np.float64), v.astype(np.float64)
    gn = torch.zeros(1, device="cuda")
    for step in (1, 2, 3):
        g = (rng.normal(size=P) * (0.3 if step != 2 else 1e-4)).astype(np.float32)
        dd.ddppo_grad_allreduce_step(ctx, cu(g), pg, mg, vg, dd.adam_cfg(step, max_grad_norm=clip),
                                     freeze_mask=cu(fr) if freeze else None, grad_norm=gn)
        po, mo, vo, n_o = optim.adam_step(po, g, mo, vo, step, max_grad_norm=clip if clip > 0 else None,
                                          freeze=fr.astype(bool) if freeze else None)
        torch.cuda.synchronize()
        assert abs(gn.item() - n_o) <= 1e-5 * n_o
    close_rel(pg.cpu().numpy() - p, po - p, 1e-4, "delta params")
    close_rel(mg.cpu().numpy(), mo, 1e-5, "m")
    close_rel(vg.cpu().numpy(), vo, 1e-5, "v")
    if freeze:
        f = fr.astype(bool)
        assert np.array_equal(pg.cpu().numpy()[f], p[f])  # bit-identical


# ------------------------------------------------------------------ a5 / a7 networks
VISUAL = {"depth": dict(obs=(1, 64, 64), layers=1), "rgbd": dict(obs=(4, 256, 256), layers=2),
          "serx50": dict(obs=(4, 256, 256), layers=2), "serx101": dict(obs=(4, 256, 256), layers=2)}


def _net_case(dd, ctx, arch, E, T, B, seed, lengths=None, hidden=None):
    desc = dd.model_desc(arch, hidden)
    H = desc.hidden
    lay = dd.param_layout(desc)
    P = dd.param_count(desc)
    params = synth.init_params([(off, int(np.prod(s)), fan) for _, off, s, fan in lay], P, seed)
    vis = VISUAL.get(arch)
    ro = synth.rollout(E, T, seed, length=lengths, hidden=H, obs_shape=vis["obs"] if vis else None,
                       rnn_layers=vis["layers"] if vis else 1)
    rng = np.random.default_rng(seed)
    env_idx = rng.permutation(E)[:B].astype(np.int32)
    L = ro["length"][env_idx]
    T_run = int(L.max())
    vo_ = {k: t.cuda() for k, t in dd.visual_obs(ro["obs"], arch in ("rgbd", "serx50", "serx101")).items()} if vis else {}
    batch = dd.make_batch(cu(ro["goal"]), cu(ro["prev_action"]), cu(ro["mask"]), cu(ro["h0"]), cu(ro["length"]),
                          cu(env_idx), E, T, ro["ld"], B, T_run, int(L.sum()),
                          obs=vo_.get("obs"), c0=cu(ro["c0"]) if vis else None, obs_rgb=vo_.get("obs_rgb"))
    ws = torch.zeros(dd.workspace_size(desc, B, T_run) // 4 + 64, device="cuda")
    lg = torch.zeros((B, T_run, 4), device="cuda")
    vl = torch.zeros((B, T_run), device="cuda")
    pg = cu(params)
    dd.ddppo_policy_fwd(ctx, desc, pg, batch, lg, vl, ws)
    dec = dd.ddppo_debug_depth_decisions(ctx, desc, batch, ws).cpu().numpy() if vis else None
    dl = rng.normal(0, 1e-2, (B, T_run, 4)).astype(np.float32)
    dv = rng.normal(0, 1e-2, (B, T_run)).astype(np.float32)
    grad = torch.full((P,), 3.0, device="cuda")
    dd.ddppo_policy_bwd(ctx, desc, pg, batch, cu(dl), cu(dv), grad, ws)
    torch.cuda.synchronize()
    ob = {"goal": ro["goal"][env_idx, :T_run], "prev_action": ro["prev_action"][env_idx, :T_run],
          "mask": ro["mask"][env_idx, :T_run], "h0": ro["h0"][env_idx]}
    if vis:
        ob.update(obs=ro["obs"][env_idx, :T_run], c0=ro["c0"][env_idx])
    lo, vo, cache = models.forward(arch, params, ob, hidden=H)
    if vis:
        _adopt_decisions(arch, params, ob, cache, dec, B * T_run, hidden=H)
    go = models.backward(arch, params, cache, dl.astype(np.float64), dv.astype(np.float64), hidden=H)
    return lay, lg.cpu().numpy(), vl.cpu().numpy(), grad.cpu().numpy(), lo, vo, go


def _adopt_decisions(arch, params, ob, cache, dec, F, tie=2.5e-4, hidden=512):
    """Hand the oracle's backward the kernel forward's ReLU masks / max-pool argmax (reading R6):
    every decision the two sides take differently must be a near-tie in the oracle's fp64
    forward (|pre-activation| <= tie * rms of its layer; pool: within tie of the window max),
    i.e. a case where both choices are correct; everything else must agree exactly.  tie = 2.5e-4
    ~ 16 * 2^-16: the forward GEMMs' bf16x3 products carry ~16-bit mantissas, summed over up to 2304
    terms and divided by the GroupNorm sigma (R6)."""
    p = models.unpack(arch, params, hidden=hidden)
    x = np.asarray(ob["obs"], np.float64).reshape((F,) + ob["obs"].shape[2:])
    enc = cache["enc"]
    off = [0]

    def take(shape_nchw):
        n = int(np.prod(shape_nchw))
        N, C, Hh, Ww = shape_nchw
        a = dec[off[0]:off[0] + n].reshape(N, Hh, Ww, C).transpose(0, 3, 1, 2)
        off[0] += n
        return a

    def adopt(key, pre):
        gpu = take(pre.shape).astype(bool)
        diff = gpu != (pre > 0)
        if diff.any():
            rms = np.sqrt(np.mean(pre ** 2))
            assert np.all(np.abs(pre[diff]) <= tie * rms), (key, np.abs(pre[diff]).max() / rms)
        enc[key] = gpu
        return pre * gpu

    def cg(z, c, g, s, pad):
        y, _ = convnets.conv_fwd(z, p[c + ".weight"], s, pad)
        return convnets.gn_fwd(y, p[g + ".weight"], p[g + ".bias"])[0]

    if arch in ("rgbd", "serx50", "serx101"):
        x = convnets.avgpool2_fwd(convnets.rgbd_normalize(x))
    z = adopt("enc.stem.conv.relu", cg(x, "enc.stem.conv", "enc.stem.gn", 2, 3))
    _, pc = convnets.maxpool_fwd(z)
    N, C, Hh, Ww = z.shape
    Ho = pc[5]
    gpu_arg = take((N, C, Ho, Ho)).astype(np.int64)
    if not np.array_equal(gpu_arg, pc[1]):
        zp = np.pad(z, ((0, 0), (0, 0), (1, 1), (1, 1)), constant_values=-np.inf)
        win = np.stack([zp[:, :, u:u + 2 * Ho:2, v:v + 2 * Ho:2] for u in range(3) for v in range(3)], axis=-1)
        picked = np.take_along_axis(win, gpu_arg[..., None], -1)[..., 0]
        d = gpu_arg != pc[1]
        assert np.all(win.max(axis=-1)[d] - picked[d] <= tie * np.sqrt(np.mean(z ** 2))), "pool argmax"
    enc["pool"] = pc[:1] + (gpu_arg,) + pc[2:]
    z, _ = convnets.maxpool_fwd(z)  # the pooled values are the same whichever tied element is picked
    cin = 32
    nblocks = {"rgbd": convnets.R50_BLOCKS, "serx50": convnets.R50_BLOCKS, "serx101": convnets.R101_BLOCKS}.get(
        arch, (2, 2, 2, 2))
    for li, (w, nb) in enumerate(zip(convnets.WIDTHS, nblocks)):
        for bi in range(nb):
            s = 2 if (bi == 0 and li > 0) else 1
            pre = f"enc.layer{li + 1}.{bi}"
            if arch in ("serx50", "serx101"):  # grouped 3x3 and squeeze-excitation before the addition (R9)
                cout = 4 * w
                a = adopt(pre + ".conv1.relu", cg(z, pre + ".conv1", pre + ".gn1", 1, 0))
                y2, _ = convnets.conv_fwd_grouped(a, p[pre + ".conv2.weight"], s, 1, convnets.SERX_CARD)
                a = adopt(pre + ".conv2.relu", convnets.gn_fwd(y2, p[pre + ".gn2.weight"], p[pre + ".gn2.bias"])[0])
                c3 = cg(a, pre + ".conv3", pre + ".gn3", 1, 0)
                b, _ = convnets.se_fwd(c3, p[pre + ".se.fc1.weight"], p[pre + ".se.fc1.bias"],
                                       p[pre + ".se.fc2.weight"], p[pre + ".se.fc2.bias"])
            elif arch == "rgbd":  # bottleneck 1x1 -> 3x3 (stride) -> 1x1
                cout = 4 * w
                a = adopt(pre + ".conv1.relu", cg(z, pre + ".conv1", pre + ".gn1", 1, 0))
                a = adopt(pre + ".conv2.relu", cg(a, pre + ".conv2", pre + ".gn2", s, 1))
                b = cg(a, pre + ".conv3", pre + ".gn3", 1, 0)
            else:
                cout = w
                a = adopt(pre + ".conv1.relu", cg(z, pre + ".conv1", pre + ".gn1", s, 1))
                b = cg(a, pre + ".conv2", pre + ".gn2", 1, 1)
            sc = cg(z, pre + ".down.conv", pre + ".down.gn", s, 0) if (s != 1 or cin != cout) else z
            z = adopt(pre + ".out", b + sc)
            cin = cout
    adopt("enc.compress.conv.relu", cg(z, "enc.compress.conv", "enc.compress.gn", 1, 1))
    vis = dec[off[0]:off[0] + F * 512].reshape(cache["vis"].shape).astype(bool)
    vpre = cache["flat"] @ p["visual_fc.weight"].T + p["visual_fc.bias"]
    d = vis != (vpre > 0)
    assert np.all(np.abs(vpre[d]) <= tie * np.sqrt(np.mean(vpre ** 2))), "visual fc relu"
    cache["vis"] = vis.astype(np.float64)  # backward only reads its > 0 mask
    off[0] += F * 512
    assert off[0] == dec.size


def test_toy_network_parity(dd, ctx):
    lay, lg, vl, g, lo, vo, go = _net_case(dd, ctx, "toy", 2, 4, 2, 11)
    close_rel(lg, lo, 1e-4, "logits")
    close_rel(vl, vo, 1e-4, "values")
    for name, off, shape, _ in lay:
        n = int(np.prod(shape))
        close_rel(g[off:off + n], go[off:off + n], 1e-4, name)


@pytest.mark.parametrize("E,T,B,lengths", [(4, 128, 2, None), (16, 128, 8, None), (4, 128, 2, [128, 40, 77, 32]),
                                           (3, 37, 3, [37, 1, 20]), (8, 300, 1, None)])
def test_gps_network_parity(dd, ctx, E, T, B, lengths):
    lay, lg, vl, g, lo, vo, go = _net_case(dd, ctx, "gps", E, T, B, 12 + E + T, lengths)
    assert rel_l2(lg, lo) < 2e-2 and rel_l2(vl, vo) < 2e-2, (rel_l2(lg, lo), rel_l2(vl, vo))
    for name, off, shape, _ in lay:
        n = int(np.prod(shape))
        e = rel_l2(g[off:off + n], go[off:off + n])
        assert e < 2e-2, (name, e)


# Depth agent (configs[2]): bf16x3 forward GEMMs, bf16 gradient GEMMs, fp16 LSTM recurrence;
# north_star's 2e-2 per-tensor relative L2 for bf16-GEMM network gradients, with the oracle's
# backward taking the kernel's ReLU / max-pool decisions where they are near-ties (reading Z24).
@pytest.mark.parametrize("E,T,B,lengths", [(2, 6, 2, [6, 3]), (3, 20, 2, [20, 7, 13]),
                                           (4, 128, 2, None),           # the config's minibatch: F = 256 frames
                                           (4, 6, 4, [6, 2, 5, 6]),      # LSTM B = 4 (16-byte exchange packets)
                                           (8, 6, 8, None),              # LSTM B = 8 (configs[4]: 16 envs / 2 minibatches)
                                           (16, 4, 8, [4, 1, 3, 4, 2, 4, 4, 1, 3, 4, 4, 2, 1, 4, 3, 4])])
def test_depth_network_parity(dd, ctx, E, T, B, lengths):
    lay, lg, vl, g, lo, vo, go = _net_case(dd, ctx, "depth", E, T, B, 40 + E + T, lengths)
    assert rel_l2(lg, lo) < 1e-3 and rel_l2(vl, vo) < 1e-3, (rel_l2(lg, lo), rel_l2(vl, vo))
    bad = []
    for name, off, shape, _ in lay:
        n = int(np.prod(shape))
        e = rel_l2(g[off:off + n], go[off:off + n])
        if not e < 2e-2:
            bad.append((name, e))
    assert not bad, bad


# NEXT-3's 1024-d LSTM (lstm_wide.cu: 32 CTAs exchanging h / partials through L2) on the
# Depth encoder (a cheap oracle), single env to eight envs per minibatch, ragged lengths
@pytest.mark.parametrize("E,T,B,lengths", [(2, 20, 2, [20, 9]), (4, 6, 4, [6, 2, 5, 6]), (8, 5, 8, None),
                                           (3, 7, 1, None)])
def test_depth_lstm1024_network_parity(dd, ctx, E, T, B, lengths):
    lay, lg, vl, g, lo, vo, go = _net_case(dd, ctx, "depth", E, T, B, 70 + E + T, lengths, hidden=1024)
    assert rel_l2(lg, lo) < 1e-3 and rel_l2(vl, vo) < 1e-3, (rel_l2(lg, lo), rel_l2(vl, vo))
    bad = []
    for name, off, shape, _ in lay:
        n = int(np.prod(shape))
        e = rel_l2(g[off:off + n], go[off:off + n])
        if not e < 2e-2:
            bad.append((name, e))
    assert not bad, bad


# RGB-D agent (configs[3]) and its SE-ResNeXt50/2 variant (NEXT-3): the same tolerances; 256x256
# frames keep the fp64 oracle to a few frames
@pytest.mark.parametrize("arch,E,T,B,lengths", [("rgbd", 2, 2, 2, [2, 1]), ("serx50", 2, 2, 2, [2, 1]),
                                                ("serx101", 2, 1, 2, None)])
def test_rgbd_network_parity(dd, ctx, arch, E, T, B, lengths):
    lay, lg, vl, g, lo, vo, go = _net_case(dd, ctx, arch, E, T, B, 60 + E + T, lengths)
    assert rel_l2(lg, lo) < 1e-3 and rel_l2(vl, vo) < 1e-3, (rel_l2(lg, lo), rel_l2(vl, vo))
    bad = []
    for name, off, shape, _ in lay:
        n = int(np.prod(shape))
        e = rel_l2(g[off:off + n], go[off:off + n])
        if not e < 2e-2:
            bad.append((name, e))
    assert not bad, bad


# ------------------------------------------------------------------ the whole learner step (a2..a8), N = 1
@pytest.mark.parametrize("cfgname,lengths", [("toy", None), ("gps", None), ("gps", [128, 96, 128, 32])])
def test_learner_step_parity(dd, ctx, cfgname, lengths):
    """ddppo_learner_step against the oracle's whole learner step (oracle/learner.py, its composition
    pinned by tests/test_oracle_nets.py).  GPS: the update's per-tensor error is bounded at 5e-2 because
    Adam's first steps are ~lr*sign(g): an element whose gradient sits within the bf16 GEMM error of 0
    may legitimately step the other way.  The factors are pinned at north_star's tolerances by
    test_learner_chain_parity (gradient 2e-2, Adam 1e-4)."""
    from paper_1911_00357_b200.learner import Learner
    c = dict(synth.CONFIGS[cfgname])
    desc = dd.model_desc(c["arch"])
    lay = dd.param_layout(desc)
    P = dd.param_count(desc)
    p0 = synth.init_params([(off, int(np.prod(s)), fan) for _, off, s, fan in lay], P, 21)
    lrn = Learner(ctx, c["arch"], c["E"], c["T"], c["epochs"], c["minibatches"], params=p0, normalize_adv=True)
    ro = synth.rollout(c["E"], c["T"], 22, length=lengths, hidden=desc.hidden)
    pm = synth.perms(22, 0, c["epochs"], c["E"])
    lrn.load_rollout(ro, pm)
    stats = lrn.step().cpu().numpy()
    torch.cuda.synchronize()
    ctx.check()
    po, mo, vo, step, info = learner.learner_step(c["arch"], p0, np.zeros(P), np.zeros(P), 0, [ro], [pm],
                                                  dict(epochs=c["epochs"], minibatches=c["minibatches"]),
                                                  hidden=desc.hidden)
    assert lrn.adam_step == step == c["epochs"] * c["minibatches"]
    A = lrn.adv.cpu().numpy()
    for n in range(c["E"]):
        close_rel(A[n, :info["adv"][0].shape[1]], info["adv"][0][n], 1e-5, "adv")
    tol = {"toy": 1e-4, "gps": 2e-2}[cfgname]
    for k, ms in enumerate(info["mb_stats"]):
        for i, name in enumerate(ppo.STAT_NAMES):
            ref = ms[name]
            assert abs(stats[k, i] - ref) <= tol * abs(ref) + tol * 1e-2, (k, name, stats[k, i], ref)
    dp = lrn.params.cpu().numpy().astype(np.float64) - p0
    dpo = po - p0
    bad = []
    for name, off, shape, _ in lay:
        n = int(np.prod(shape))
        e = rel_l2(dp[off:off + n], dpo[off:off + n])
        if not e < (1e-3 if cfgname == "toy" else 5e-2):
            bad.append((name, round(e, 4)))
    assert not bad, bad


@pytest.mark.parametrize("cfgname,T,lengths,frozen,replay", [("gps", 128, [128, 96, 128, 32], False, False),
                                                             ("depth", 12, [12, 5, 12, 9], False, False),
                                                             ("depth", 128, [128, 128, 70, 128], False, False),
                                                             ("rgbd", 2, [2, 1, 2, 2], False, False),
                                                             ("depth", 12, [12, 5, 12, 9], True, False),
                                                             ("rgbd", 2, [2, 1, 2, 2], True, False),
                                                             ("serx50", 2, [2, 1, 2, 2], False, False),
                                                             # logp_old / V_old from a replay
                                                             # forward of theta -> rho = 1 at minibatch 1
                                                             ("gps", 128, [128, 96, 128, 32], False, True),
                                                             ("depth", 12, [12, 5, 12, 9], False, True)])
def test_learner_chain_parity(dd, ctx, cfgname, T, lengths, frozen, replay):
    """The learner step of the config (Adam eps 1e-8, 2 epochs x 2 minibatches) driven one ABI call
    at a time -- ddppo_gae, ddppo_adv_norm, then per minibatch ddppo_policy_fwd,
    ddppo_ppo_loss_grad, ddppo_policy_bwd, ddppo_grad_allreduce_step -- each minibatch checked
    against the oracle evaluated at the kernels' own parameters for that minibatch, with the
    kernels' ReLU / max-pool decisions handed over (reading R6):
      GAE / normalisation statistics 1e-5; logits / values; loss statistics; every parameter
      tensor's gradient within north_star's 2e-2 relative L2; the clip + Adam update of that
      gradient 1e-4 (m, v 1e-5).
    Then ddppo_learner_step on the same rollout must reproduce the chained calls' parameters
    (the visual agents: bit for bit -- the same kernels in the same order; GPS: its learner fuses
    head + loss into the recurrence epilogue, so to 1e-3 of the update).
    frozen: the transfer setting of P:L407 (NEXT-4) -- a frozen visual encoder: no encoder backward
    (its gradient exactly 0), its parameters bit-identical through the step."""
    from paper_1911_00357_b200.learner import Learner
    c = dict(synth.CONFIGS[cfgname])
    c["T"] = T
    E, ep, mb = c["E"], c["epochs"], c["minibatches"]
    B = E // mb
    desc = dd.model_desc(c["arch"])
    H = desc.hidden
    lay = dd.param_layout(desc)
    P = dd.param_count(desc)
    p0 = synth.init_params([(off, int(np.prod(s)), fan) for _, off, s, fan in lay], P, 23)
    ro = synth.rollout(E, T, 24, length=lengths, hidden=H, obs_shape=c.get("obs"), rnn_layers=c.get("rnn_layers", 1))
    if replay:  # the behaviour policy is theta itself: log pi_theta(a|s) and V_theta(s) from the oracle
        ob = {k: ro[k] for k in ("goal", "prev_action", "mask", "h0")}
        if "obs" in ro:
            ob.update(obs=ro["obs"], c0=ro["c0"])
        ob["prev_action"] = ro["prev_action"][:, :T]
        ob["mask"] = ro["mask"][:, :T]
        lo, vo, _ = models.forward(c["arch"], p0, ob, hidden=H)
        logp = lo - np.log(np.exp(lo - lo.max(-1, keepdims=True)).sum(-1, keepdims=True)) - lo.max(-1, keepdims=True)
        a = ro["action"][:, :T]
        ro["logp_old"][:, :T] = np.take_along_axis(logp, a[..., None].astype(np.int64), -1)[..., 0]
        ro["val"][:, :T] = vo
    pm = synth.perms(24, 0, ep, E)
    ld = ro["ld"]
    vis = c["arch"] in ("depth", "rgbd", "serx50")
    g = {k: cu(ro[k]) for k in ("rew", "val", "goal", "mask", "logp_old", "h0")}
    for k in ("prev_action", "action", "length"):
        g[k] = torch.from_numpy(np.ascontiguousarray(ro[k])).cuda()
    g["done"] = torch.from_numpy(np.ascontiguousarray(ro["done"])).cuda()
    if vis:
        g.update({k: t.cuda() for k, t in dd.visual_obs(ro["obs"], c["arch"] in ("rgbd", "serx50")).items()})
        g["c0"] = cu(ro["c0"])
    adv, ret = torch.zeros((E, ld), device="cuda"), torch.zeros((E, ld), device="cuda")
    stats3 = torch.zeros(4, dtype=torch.float64, device="cuda")
    mis = torch.zeros(4, device="cuda")
    dd.ddppo_gae(ctx, g["rew"], g["val"], g["done"], g["length"], E, T, ld, 0.99, 0.95, adv, ret, stats3)
    dd.ddppo_adv_norm(ctx, stats3, 1e-5, mis)
    # oracle a2 / a3
    from oracle import advnorm, gae as ogae
    a_o, r_o = ogae.gae(ro["rew"], ro["val"], ro["done"], ro["length"], 0.99, 0.95)
    Tm = a_o.shape[1]
    a_o = np.pad(a_o, ((0, 0), (0, T - Tm)))
    r_o = np.pad(r_o, ((0, 0), (0, T - Tm)))
    mis_o = advnorm.mean_invstd(ogae.adv_stats(a_o, ro["length"]), 1e-5)
    torch.cuda.synchronize()
    close_rel(adv.cpu().numpy()[:, :T], a_o, 1e-5, "adv")
    m_gpu = mis.cpu().numpy()
    assert abs(m_gpu[0] - mis_o[0]) <= 1e-5 * abs(mis_o[0]) + 1e-6 and abs(m_gpu[1] - mis_o[1]) <= 1e-5 * mis_o[1]
    params = cu(p0)
    m, v = torch.zeros(P, device="cuda"), torch.zeros(P, device="cuda")
    lcfg = dd.loss_cfg(normalize_adv=True)
    cfg_o = dict(learner.DEFAULT_CFG, epochs=ep, minibatches=mb, freeze_encoder=frozen)
    from oracle import transfer
    enc = transfer.encoder_mask(c["arch"], P) if frozen else None
    fmask = torch.from_numpy(enc.astype(np.uint8)).cuda() if frozen else None
    k = 0
    for e in range(ep):
        for j in range(mb):
            envs = pm[e][j * B:(j + 1) * B]
            L = ro["length"][envs]
            T_run = int(L.max())
            F = B * T_run
            env_idx = torch.from_numpy(np.ascontiguousarray(envs.astype(np.int32))).cuda()
            batch = dd.make_batch(g["goal"], g["prev_action"], g["mask"], g["h0"], g["length"], env_idx, E, T, ld, B,
                                  T_run, int(L.sum()), obs=g.get("obs"), c0=g.get("c0"), obs_rgb=g.get("obs_rgb"),
                                  freeze_encoder=frozen)
            ws = torch.zeros(dd.workspace_size(desc, B, T_run) // 4 + 64, device="cuda")
            lg, vl = torch.zeros((B, T_run, 4), device="cuda"), torch.zeros((B, T_run), device="cuda")
            dlg, dvl = torch.zeros_like(lg), torch.zeros_like(vl)
            st = torch.zeros(8, device="cuda")
            grad = torch.full((P,), 3.0, device="cuda")
            theta = params.cpu().numpy().astype(np.float64)
            m_k, v_k = m.cpu().numpy().astype(np.float64), v.cpu().numpy().astype(np.float64)
            dd.ddppo_policy_fwd(ctx, desc, params, batch, lg, vl, ws)
            dec = dd.ddppo_debug_depth_decisions(ctx, desc, batch, ws).cpu().numpy() if vis else None
            dd.ddppo_ppo_loss_grad(ctx, lg, vl, batch, g["action"], g["logp_old"], g["val"], ret, adv, mis, lcfg,
                                   dlg, dvl, st)
            dd.ddppo_policy_bwd(ctx, desc, params, batch, dlg, dvl, grad, ws)
            torch.cuda.synchronize()
            g_k = grad.cpu().numpy().astype(np.float64)
            if frozen:
                assert np.all(g_k[enc] == 0), k
            dd.ddppo_grad_allreduce_step(ctx, grad, params, m, v, dd.adam_cfg(k + 1), freeze_mask=fmask)
            torch.cuda.synchronize()
            ctx.check()
            # the oracle at the kernels' parameters theta_k, with their decisions
            hook = (lambda b_, c_: _adopt_decisions(c["arch"], theta, b_, c_, dec, F)) if vis else None
            go, so, (lo, vo, _, _) = learner.minibatch_grad(c["arch"], theta, ro, a_o, r_o, envs, mis_o, cfg_o,
                                                            hidden=H, adopt=hook)
            lim = 1e-3 if vis else 2e-2
            assert rel_l2(lg.cpu().numpy(), lo) < lim and rel_l2(vl.cpu().numpy(), vo) < lim, k
            sg = st.cpu().numpy()
            for i, name in enumerate(ppo.STAT_NAMES):
                assert abs(sg[i] - so[name]) <= 2e-2 * abs(so[name]) + 2e-4, (k, name, sg[i], so[name])
            bad = []
            for name, off, shape, _ in lay:
                n = int(np.prod(shape))
                e_ = rel_l2(g_k[off:off + n], go[off:off + n])
                if not e_ < 2e-2:
                    bad.append((name, e_))
            assert not bad, (k, bad)
            # a8 (N = 1): clip + Adam of the kernels' gradient
            p_o, mm_o, vv_o, _ = optim.adam_step(theta, g_k, m_k, v_k, k + 1, freeze=enc)
            close_update(params.cpu().numpy(), theta, p_o, 1e-4, f"update {k}")
            close_rel(m.cpu().numpy(), mm_o, 1e-5, f"m {k}")
            close_rel(v.cpu().numpy(), vv_o, 1e-5, f"v {k}")
            k += 1
    chain = params.cpu().numpy()
    if frozen:
        assert np.array_equal(chain[enc], p0[enc])
    # the same step through ddppo_learner_step (graph-captured on its second use: run it twice)
    for it in range(2):
        lrn = Learner(ctx, c["arch"], E, T, ep, mb, params=p0, normalize_adv=True, freeze_encoder=frozen)
        lrn.load_rollout(ro, pm)
        lrn.step()
        torch.cuda.synchronize()
        ctx.check()
        got = lrn.params.cpu().numpy()
        if vis:
            assert np.array_equal(got, chain), (it, np.abs(got - chain).max())
        else:
            assert rel_l2(got - p0, chain - p0) < 1e-3, it


# ------------------------------------------------------------------ CUDA-graph replay of the learner step
@pytest.mark.parametrize("cfgname,hidden", [("gps", None), ("toy", None), ("depth", None), ("depth", 1024)])
def test_learner_graph_replay_matches_eager(dd, ctx, cfgname, hidden):
    """Three learner steps: eager (graphs off) vs captured-and-replayed (the second step is captured,
    the third replays) -- the parameters, Adam moments and loss statistics agree bit for bit.  Depth
    with the 1024-d LSTM: the 32-CTA recurrences' L2 exchange (counters reset in the graph) replays
    deterministically too."""
    from paper_1911_00357_b200.learner import Learner
    c = dict(synth.CONFIGS[cfgname])
    if cfgname == "depth":
        c.update(T=16)  # a short rollout keeps the test fast; the path is the config's
    desc = dd.model_desc(c["arch"], hidden)
    lay = dd.param_layout(desc)
    P = dd.param_count(desc)
    p0 = synth.init_params([(off, int(np.prod(s)), fan) for _, off, s, fan in lay], P, 31)
    out = {}
    for graphs in (False, True):
        dd.ddppo_set_graphs(ctx, graphs)
        lrn = Learner(ctx, c["arch"], c["E"], c["T"], c["epochs"], c["minibatches"], hidden=desc.hidden, params=p0,
                      normalize_adv=True)
        for it in range(3):
            ro = synth.rollout(c["E"], c["T"], 32, iteration=it, hidden=desc.hidden, obs_shape=c.get("obs"),
                               rnn_layers=c.get("rnn_layers", 1))
            lrn.load_rollout(ro, synth.perms(32, it, c["epochs"], c["E"]))
            lrn.step()
        torch.cuda.synchronize()
        ctx.check()
        out[graphs] = (lrn.params.cpu().numpy(), lrn.m.cpu().numpy(), lrn.v.cpu().numpy(), lrn.stats.cpu().numpy(),
                       lrn.adam_step)
    dd.ddppo_set_graphs(ctx, True)
    for a, b in zip(out[False], out[True]):
        assert np.array_equal(np.asarray(a), np.asarray(b))


@pytest.mark.gpu
def test_learner_graph_alternating_stats_buffers(dd, ctx):
    """Double-buffered statistics (the pipelined training loop): the two keys alternate, each is
    captured on its second use and replayed after -- five steps agree bit for bit with eager."""
    from paper_1911_00357_b200.learner import Learner
    c = synth.CONFIGS["gps"]
    desc = dd.model_desc(c["arch"])
    lay = dd.param_layout(desc)
    P = dd.param_count(desc)
    p0 = synth.init_params([(off, int(np.prod(s)), fan) for _, off, s, fan in lay], P, 41)
    out = {}
    for graphs in (False, True):
        dd.ddppo_set_graphs(ctx, graphs)
        lrn = Learner(ctx, c["arch"], c["E"], c["T"], c["epochs"], c["minibatches"], params=p0, normalize_adv=True)
        bufs = [torch.zeros_like(lrn.stats) for _ in range(2)]
        rec = []
        for it in range(5):
            ro = synth.rollout(c["E"], c["T"], 42, iteration=it, hidden=desc.hidden)
            lrn.load_rollout(ro, synth.perms(42, it, c["epochs"], c["E"]))
            lrn.step(stats=bufs[it % 2])
            torch.cuda.synchronize()
            rec.append(bufs[it % 2].cpu().numpy().copy())
        ctx.check()
        out[graphs] = (lrn.params.cpu().numpy(), np.stack(rec))
    dd.ddppo_set_graphs(ctx, True)
    for a, b in zip(out[False], out[True]):
        assert np.array_equal(a, b)
