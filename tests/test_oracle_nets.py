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


def test_learner_equal_buffers_two_ranks_equals_one_rank_and_equal_weighting():
    """N=2 with identical buffers == N=1; unequal lengths -> mean of per-rank grads."""
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
