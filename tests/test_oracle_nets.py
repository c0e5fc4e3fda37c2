"""Pins for oracle.nets / oracle.models / oracle.learner (steps a5, a7, a8 composition)."""
import numpy as np
import torch

import synth
from oracle import learner, models, nets, ppo



def _t(a):
    return torch.tensor(np.asarray(a, dtype=np.float64))


def test_gru_matches_torch_grucell_with_masks():
    rng = np.random.default_rng(0)
    B, T, I, H = 3, 9, 5, 7
    cell = torch.nn.GRUCell(I, H).double()
    W_ih, W_hh = cell.weight_ih.detach().numpy(), cell.weight_hh.detach().numpy()
    b_ih, b_hh = cell.bias_ih.detach().numpy(), cell.bias_hh.detach().numpy()
    x = rng.normal(size=(B, T, I))
    mask = (rng.random((B, T)) > 0.2).astype(float)
    h0 = rng.normal(size=(B, H))
    dh_out = rng.normal(size=(B, T, H))
    h, cache = nets.gru_seq_fwd(x, mask, h0, W_ih, W_hh, b_ih, b_hh)
    xt = _t(x).requires_grad_(True)
    hp = _t(h0)
    outs = []
    for t in range(T):
        hp = cell(xt[:, t], _t(mask[:, t:t + 1]) * hp)
        outs.append(hp)
    ht = torch.stack(outs, 1)
    assert np.max(np.abs(ht.detach().numpy() - h)) < 1e-13
    (ht * _t(dh_out)).sum().backward()
    dx, dWi, dWh, dbi, dbh = nets.gru_seq_bwd(dh_out, cache, W_ih, W_hh)
    for mine, ref in ((dx, xt.grad), (dWi, cell.weight_ih.grad), (dWh, cell.weight_hh.grad),
                      (dbi, cell.bias_ih.grad), (dbh, cell.bias_hh.grad)):
        assert np.max(np.abs(mine - ref.numpy())) < 1e-12


def test_lstm_matches_torch_lstmcell_with_masks():
    rng = np.random.default_rng(1)
    B, T, I, H = 2, 8, 4, 6
    cell = torch.nn.LSTMCell(I, H).double()
    W_ih, W_hh = cell.weight_ih.detach().numpy(), cell.weight_hh.detach().numpy()
    b_ih, b_hh = cell.bias_ih.detach().numpy(), cell.bias_hh.detach().numpy()
    x = rng.normal(size=(B, T, I))
    mask = (rng.random((B, T)) > 0.3).astype(float)
    h0, c0 = rng.normal(size=(B, H)), rng.normal(size=(B, H))
    dh_out = rng.normal(size=(B, T, H))
    h, cache = nets.lstm_seq_fwd(x, mask, h0, c0, W_ih, W_hh, b_ih, b_hh)
    xt = _t(x).requires_grad_(True)
    hp, cp = _t(h0), _t(c0)
    outs = []
    for t in range(T):
        m = _t(mask[:, t:t + 1])
        hp, cp = cell(xt[:, t], (m * hp, m * cp))
        outs.append(hp)
    ht = torch.stack(outs, 1)
    assert np.max(np.abs(ht.detach().numpy() - h)) < 1e-13
    (ht * _t(dh_out)).sum().backward()
    dx, dWi, dWh, dbi, dbh = nets.lstm_seq_bwd(dh_out, cache, W_ih, W_hh)
    for mine, ref in ((dx, xt.grad), (dWi, cell.weight_ih.grad), (dWh, cell.weight_hh.grad),
                      (dbi, cell.bias_ih.grad), (dbh, cell.bias_hh.grad)):
        assert np.max(np.abs(mine - ref.numpy())) < 1e-12


def test_zero_whh_reduces_gru_to_feedforward():
    rng = np.random.default_rng(2)
    B, T, I, H = 2, 4, 3, 5
    W_ih, b_ih, b_hh = rng.normal(size=(3 * H, I)), rng.normal(size=3 * H), rng.normal(size=3 * H)
    x = rng.normal(size=(B, T, I))
    h, _ = nets.gru_seq_fwd(x, np.zeros((B, T)), np.zeros((B, H)), W_ih, np.zeros((3 * H, H)), b_ih, b_hh)
    gi = x @ W_ih.T + b_ih
    r = nets.sigmoid(gi[..., :H] + b_hh[:H])
    z = nets.sigmoid(gi[..., H:2 * H] + b_hh[H:2 * H])
    n = np.tanh(gi[..., 2 * H:] + r * b_hh[2 * H:])
    assert np.max(np.abs(h - (1 - z) * n)) < 1e-14


def _entries(arch, hidden):
    offs, P = models.offsets(arch, hidden=hidden)
    fans = {n: f for n, _, f in models.layout(arch, hidden=hidden)}
    return [(o, int(np.prod(s)), fans[k]) for k, (o, s) in offs.items()], P


def test_layout_sizes():
    assert models.offsets("toy")[1] == 581
    assert models.offsets("gps")[1] == 890661


def test_zero_params_zero_outputs():
    ro = synth.rollout(2, 6, 0, hidden=16)
    batch = {"goal": ro["goal"], "prev_action": ro["prev_action"][:, :6], "mask": ro["mask"][:, :6], "h0": ro["h0"]}
    for arch, hid in (("toy", 64), ("gps", 16)):
        P = models.offsets(arch, hidden=hid)[1]
        lg, v, _ = models.forward(arch, np.zeros(P), batch if arch == "gps" else {"goal": ro["goal"]}, hidden=hid)
        assert not lg.any() and not v.any()


def _model_loss(arch, flat, batch, lin, hidden):
    lg, v, cache = models.forward(arch, flat, batch, hidden=hidden)
    B, T = v.shape
    st, dl, dv = ppo.loss_and_grad(lg.reshape(B * T, -1), v.reshape(-1), lin["actions"], lin["logp_old"],
                                   lin["values_old"], lin["returns"], lin["adv"], np.ones(B * T, bool))
    return st["total"], cache, dl.reshape(B, T, -1), dv.reshape(B, T)


def test_model_gradients_finite_differences_and_torch():
    H = 6
    ro = synth.rollout(2, 5, 3, hidden=H)
    batch = {"goal": ro["goal"].astype(float), "prev_action": ro["prev_action"][:, :5],
             "mask": ro["mask"][:, :5].astype(float), "h0": ro["h0"].astype(float)}
    lin = {k: v.astype(np.float64) if v.dtype != np.int32 else v for k, v in synth.random_loss_inputs(10, 4).items()}
    for arch in ("toy", "gps"):
        ent, P = _entries(arch, H)
        flat = synth.init_params(ent, P, 5).astype(np.float64)
        L, cache, dl, dv = _model_loss(arch, flat, batch, lin, H)
        g = models.backward(arch, flat, cache, dl, dv, hidden=H)
        h = 1e-5
        idx = np.random.default_rng(6).choice(P, 60, replace=False)
        for i in idx:
            fp, fm = flat.copy(), flat.copy()
            fp[i] += h
            fm[i] -= h
            fd = (_model_loss(arch, fp, batch, lin, H)[0] - _model_loss(arch, fm, batch, lin, H)[0]) / (2 * h)
            assert abs(fd - g[i]) < 1e-7 * max(1.0, abs(fd)), (arch, i, fd, g[i])


def test_learner_equal_buffers_two_ranks_equals_one_rank():
    """N=2 with identical buffers == N=1.  The weighting itself is pinned by
    test_learner_composition_matches_torch_ddp_objective."""
    H = 8
    ent, P = _entries("gps", H)
    p0 = synth.init_params(ent, P, 0)
    ro = synth.rollout(4, 12, 1, hidden=H)
    pm = synth.perms(0, 0, 2, 4)
    cfg = dict(normalize_adv=False)
    a = learner.learner_step("gps", p0, np.zeros(P), np.zeros(P), 0, [ro], [pm], cfg, hidden=H)
    b = learner.learner_step("gps", p0, np.zeros(P), np.zeros(P), 0, [ro, ro], [pm, pm], cfg, hidden=H)
    assert np.max(np.abs(a[0] - b[0])) < 1e-15
    ro2 = synth.rollout(4, 12, 2, hidden=H, length=3)
    tr = []
    learner.learner_step("gps", p0, np.zeros(P), np.zeros(P), 0, [ro, ro2], [pm, pm], dict(epochs=1, minibatches=1),
                         hidden=H, trace=tr)
    # both ranks' grads are computed at the same params; the update used their plain mean
    assert tr[0]["rank"] == 0 and tr[1]["rank"] == 1
    assert np.array_equal(tr[0]["params"], tr[1]["params"])


def _torch_ppo_mean(z, v, act, lpo, vo, R, A, eps=0.2, c_v=0.5, c_e=0.01):
    """Eq. 2 + Z3/Z4 written in torch: the per-worker mean over its valid samples."""
    logp = torch.log_softmax(z, dim=1)
    lp = logp.gather(1, act[:, None])[:, 0]
    rho = torch.exp(lp - lpo)
    surr = torch.minimum(rho * A, torch.clamp(rho, 1 - eps, 1 + eps) * A)
    vc = vo + torch.clamp(v - vo, -eps, eps)
    lv = 0.5 * torch.maximum((v - R) ** 2, (vc - R) ** 2)
    ent = -(logp.exp() * logp).sum(1)
    return -surr.mean() + c_v * lv.mean() - c_e * ent.mean()


def test_learner_composition_matches_torch_ddp_objective():
    """Pins oracle.learner_step's cross-rank composition against an independent torch construction:
    toy actor-critic (R2) built from torch.nn.Linear, the DD-PPO objective (1/N) sum_r mean_r(loss)
    (P:L171 equal worker weighting; Eq. 3/4 gradient mean), advantages normalised with statistics
    of the concatenated valid entries of all ranks (Z2, torch.std unbiased), global-norm clip 0.5 on
    the averaged gradient (Z15, torch.nn.utils.clip_grad_norm_), torch.optim.Adam (Z14) stepping
    once per minibatch.  Unequal lengths (12 vs 5) make per-sample and per-rank weighting differ;
    two minibatches x two epochs exercise the Adam step index."""
    E, T = 4, 12
    ent, P = _entries("toy", 512)
    p0 = synth.init_params(ent, P, 11)
    ros = [synth.rollout(E, T, 21, rank=0, hidden=8), synth.rollout(E, T, 21, rank=1, hidden=8, length=[5, 12, 3, 7])]
    pms = [synth.perms(4, 0, 2, E, rank=r) for r in range(2)]
    po, _, _, step, info = learner.learner_step("toy", p0, np.zeros(P), np.zeros(P), 0, ros, pms, dict(epochs=2),
                                                hidden=8)
    assert step == 4
    # global advantage statistics == one rank holding the concatenation of every valid entry (Z2)
    from oracle import gae as ogae
    advs = [ogae.gae(ro["rew"], ro["val"], ro["done"], ro["length"], 0.99, 0.95) for ro in ros]
    cat = np.concatenate([a[np.arange(a.shape[1])[None, :] < np.asarray(ro["length"])[:, None]]
                          for (a, _), ro in zip(advs, ros)])
    assert info["adv_stats"][2] == cat.size == 12 * 4 + 5 + 12 + 3 + 7
    ct = torch.tensor(cat)
    mu, sd = float(ct.mean()), float(ct.std(unbiased=True))
    assert abs(info["mean_invstd"][0] - mu) < 1e-12 and abs(1.0 / info["mean_invstd"][1] - (sd + 1e-5)) < 1e-12
    # the torch DD-PPO learner
    fc1, head = torch.nn.Linear(3, 64).double(), torch.nn.Linear(64, 5).double()
    lay = {n: (off, shape) for (n, shape, _), off in zip(models.layout("toy"), [e[0] for e in ent])}
    with torch.no_grad():
        for mod, pre in ((fc1, "fc1"), (head, "head")):
            for attr in ("weight", "bias"):
                off, shape = lay[pre + "." + attr]
                getattr(mod, attr).copy_(_t(p0[off:off + int(np.prod(shape))].reshape(shape)))
    prm = list(fc1.parameters()) + list(head.parameters())
    opt = torch.optim.Adam(prm, lr=2.5e-4, betas=(0.9, 0.999), eps=1e-8)
    for e in range(2):
        for j in range(2):
            opt.zero_grad()
            tot = 0.0
            for r, ro in enumerate(ros):
                envs = pms[r][e][j * 2:(j + 1) * 2]
                sel = [(n, t) for n in envs for t in range(int(ro["length"][n]))]
                ni, ti = np.array([s[0] for s in sel]), np.array([s[1] for s in sel])
                out = head(torch.tanh(fc1(_t(ro["goal"][ni, ti]))))
                A, R = advs[r]
                An = (_t(A[ni, ti]) - mu) / (sd + 1e-5)
                tot = tot + _torch_ppo_mean(out[:, :4], out[:, 4], torch.tensor(ro["action"][ni, ti].astype(np.int64)),
                                            _t(ro["logp_old"][ni, ti]), _t(ro["val"][ni, ti]), _t(R[ni, ti]), An)
            (tot / 2).backward()
            torch.nn.utils.clip_grad_norm_(prm, 0.5)
            opt.step()
    mine = {n: po[off:off + int(np.prod(s))].reshape(s) for n, (off, s) in lay.items()}
    for mod, pre in ((fc1, "fc1"), (head, "head")):
        for attr in ("weight", "bias"):
            ref = getattr(mod, attr).detach().numpy()
            d = mine[pre + "." + attr] - ref
            assert np.max(np.abs(d)) < 1e-10, (pre, attr, np.max(np.abs(d)))
    # and the update is not trivially zero
    assert np.max(np.abs(po - p0)) > 1e-4
