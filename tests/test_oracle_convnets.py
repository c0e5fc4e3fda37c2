"""Pins for oracle.convnets and the Depth model (steps a5/a7 for configs[2]):
torch.nn.functional fp64 forward + autograd for every layer, special-case identities, and finite
differences through the whole Depth actor-critic."""
import numpy as np
import pytest
import torch
import torch.nn.functional as F

import synth
from oracle import convnets, models, ppo


def _t(a, grad=False):
    t = torch.tensor(np.asarray(a, dtype=np.float64))
    return t.requires_grad_(grad)


@pytest.mark.parametrize("k,s,p", [(3, 1, 1), (3, 2, 1), (1, 2, 0), (7, 2, 3), (1, 1, 0)])
def test_conv_matches_torch(k, s, p):
    rng = np.random.default_rng(k * 10 + s)
    x = rng.normal(size=(2, 3, 9, 10))
    W = rng.normal(size=(4, 3, k, k))
    y, cache = convnets.conv_fwd(x, W, s, p)
    xt, Wt = _t(x, True), _t(W, True)
    yt = F.conv2d(xt, Wt, stride=s, padding=p)
    assert np.max(np.abs(y - yt.detach().numpy())) < 1e-12
    dy = rng.normal(size=y.shape)
    (yt * _t(dy)).sum().backward()
    dx, dW = convnets.conv_bwd(dy, W, s, p, cache)
    assert np.max(np.abs(dx - xt.grad.numpy())) < 1e-12
    assert np.max(np.abs(dW - Wt.grad.numpy())) < 1e-12


def test_1x1_conv_is_gemm():
    rng = np.random.default_rng(0)
    x = rng.normal(size=(2, 5, 4, 4))
    W = rng.normal(size=(3, 5, 1, 1))
    y, _ = convnets.conv_fwd(x, W, 1, 0)
    ref = np.einsum("oc,nchw->nohw", W[:, :, 0, 0], x)
    assert np.max(np.abs(y - ref)) < 1e-12


@pytest.mark.parametrize("G", [1, 4, 16])
def test_groupnorm_matches_torch(G):
    rng = np.random.default_rng(G)
    x = rng.normal(size=(3, 16, 5, 6)) * 3 + 1
    gamma, beta = rng.normal(size=16), rng.normal(size=16)
    y, cache = convnets.gn_fwd(x, gamma, beta, G)
    xt, gt, bt = _t(x, True), _t(gamma, True), _t(beta, True)
    yt = F.group_norm(xt, G, gt, bt, eps=1e-5)
    assert np.max(np.abs(y - yt.detach().numpy())) < 1e-12
    dy = rng.normal(size=y.shape)
    (yt * _t(dy)).sum().backward()
    dx, dg, db = convnets.gn_bwd(dy, gamma, cache)
    for mine, ref in ((dx, xt.grad), (dg, gt.grad), (db, bt.grad)):
        assert np.max(np.abs(mine - ref.numpy())) < 1e-11


def test_groupnorm_special_cases():
    rng = np.random.default_rng(1)
    x = rng.normal(size=(2, 8, 3, 3))
    one, zero = np.ones(8), np.zeros(8)
    y_in, _ = convnets.gn_fwd(x, one, zero, G=8)  # G = C: instance norm
    m = x.mean(axis=(2, 3), keepdims=True)
    v = x.var(axis=(2, 3), keepdims=True)
    assert np.max(np.abs(y_in - (x - m) / np.sqrt(v + 1e-5))) < 1e-12
    y_ln, _ = convnets.gn_fwd(x, one, zero, G=1)  # G = 1: layer norm over (C, H, W)
    m = x.mean(axis=(1, 2, 3), keepdims=True)
    v = x.var(axis=(1, 2, 3), keepdims=True)
    assert np.max(np.abs(y_ln - (x - m) / np.sqrt(v + 1e-5))) < 1e-12


def test_maxpool_matches_torch_including_ties():
    rng = np.random.default_rng(2)
    x = np.maximum(rng.normal(size=(2, 3, 9, 8)), 0.0)  # ReLU zeros create ties
    y, cache = convnets.maxpool_fwd(x)
    xt = _t(x, True)
    yt = F.max_pool2d(xt, 3, 2, 1)
    assert np.max(np.abs(y - yt.detach().numpy())) < 1e-15
    dy = rng.normal(size=y.shape)
    (yt * _t(dy)).sum().backward()
    assert np.max(np.abs(convnets.maxpool_bwd(dy, cache) - xt.grad.numpy())) < 1e-12


class _TorchR18H(torch.nn.Module):
    """Independent torch.nn construction of the half-width ResNet18 (test-only reference)."""

    def __init__(self, p):
        super().__init__()
        self.p = p

    def forward(self, x):
        p = self.p

        def cg(z, c, g, s, pad, relu):
            z = F.conv2d(z, p[c + ".weight"], stride=s, padding=pad)
            z = F.group_norm(z, 16, p[g + ".weight"], p[g + ".bias"], eps=1e-5)
            return F.relu(z) if relu else z
        z = cg(x, "enc.stem.conv", "enc.stem.gn", 2, 3, True)
        z = F.max_pool2d(z, 3, 2, 1)
        cin = 32
        for li, c in enumerate(convnets.WIDTHS):
            for bi in range(2):
                s = 2 if (bi == 0 and li > 0) else 1
                pre = f"enc.layer{li + 1}.{bi}"
                a = cg(z, pre + ".conv1", pre + ".gn1", s, 1, True)
                b = cg(a, pre + ".conv2", pre + ".gn2", 1, 1, False)
                sc = cg(z, pre + ".down.conv", pre + ".down.gn", s, 0, False) if (s != 1 or cin != c) else z
                z = F.relu(b + sc)
                cin = c
        return cg(z, "enc.compress.conv", "enc.compress.gn", 1, 1, True)


def test_resnet18h_matches_torch():
    lay = models.layout("depth")
    offs, P = models.offsets("depth")
    ent = [(offs[n][0], int(np.prod(s)), f) for n, s, f in lay]
    flat = synth.init_params(ent, P, 3).astype(np.float64)
    rng = np.random.default_rng(4)
    flat += rng.normal(0, 0.05, P) * (np.array([1.0]))  # perturb GN affine away from (1, 0)
    p = models.unpack("depth", flat)
    x = synth.depth_frames(rng, 1, 2)[0].astype(np.float64)  # [2][1][64][64]
    feat, caches = convnets.resnet18h_fwd(x, p)
    assert feat.shape == (2, 128, 2, 2)
    pt = {k: _t(v, True) for k, v in p.items() if k.startswith("enc.")}
    xt = _t(x, True)
    ft = _TorchR18H(pt)(xt)
    assert np.max(np.abs(feat - ft.detach().numpy())) < 1e-10
    dz = rng.normal(size=feat.shape)
    (ft * _t(dz)).sum().backward()
    g = {}
    dx = convnets.resnet18h_bwd(dz, p, caches, g)
    assert np.max(np.abs(dx - xt.grad.numpy())) < 1e-9
    for k, v in pt.items():
        assert np.max(np.abs(g[k] - v.grad.numpy())) < 1e-9 * max(1.0, np.abs(v.grad.numpy()).max()), k


def test_depth_layout_size():
    assert models.offsets("depth")[1] == 5588741


def test_depth_model_finite_differences():
    lay = models.layout("depth")
    offs, P = models.offsets("depth")
    ent = [(offs[n][0], int(np.prod(s)), f) for n, s, f in lay]
    flat = synth.init_params(ent, P, 5).astype(np.float64)
    ro = synth.rollout(1, 3, 5, obs_shape=(1, 64, 64))
    batch = {k: ro[k][:, :3] for k in ("goal", "prev_action", "mask")}
    batch.update(obs=ro["obs"], h0=ro["h0"], c0=ro["c0"])
    lin = {k: v.astype(np.float64) if v.dtype != np.int32 else v for k, v in synth.random_loss_inputs(3, 6).items()}

    def loss(fl):
        lg, v, cache = models.forward("depth", fl, batch)
        st, dl, dv = ppo.loss_and_grad(lg.reshape(3, -1), v.reshape(-1), lin["actions"], lin["logp_old"],
                                       lin["values_old"], lin["returns"], lin["adv"], np.ones(3, bool))
        return st["total"], cache, dl.reshape(1, 3, -1), dv.reshape(1, 3)

    L, cache, dl, dv = loss(flat)
    g = models.backward("depth", flat, cache, dl, dv)
    rng = np.random.default_rng(7)
    names = ["enc.stem.conv.weight", "enc.layer2.0.down.conv.weight", "enc.layer4.1.gn2.weight",
             "enc.compress.conv.weight", "visual_fc.weight", "rnn.weight_ih", "rnn.weight_hh", "goal_fc.weight"]
    for name in names:
        o, s = offs[name]
        for i in rng.choice(int(np.prod(s)), 3, replace=False):
            fp, fm = flat.copy(), flat.copy()
            fp[o + i] += 1e-7
            fm[o + i] -= 1e-7
            fd = (loss(fp)[0] - loss(fm)[0]) / 2e-7
            # ReLU / max-pool kinks can sit inside the stencil: 1e-4 relative (the exact layer-by-layer
            # pins are the torch.autograd cross-checks above)
            assert abs(fd - g[o + i]) < 1e-4 * max(abs(fd), 1e-3), (name, i, fd, g[o + i])


# ---------------------------------------------------------------- RGB-D agent (configs[3])
def test_avgpool_matches_torch():
    rng = np.random.default_rng(9)
    x = rng.normal(size=(2, 3, 8, 6))
    xt = _t(x, True)
    yt = F.avg_pool2d(xt, 2, 2)
    assert np.max(np.abs(convnets.avgpool2_fwd(x) - yt.detach().numpy())) < 1e-14
    dy = rng.normal(size=yt.shape)
    (yt * _t(dy)).sum().backward()
    assert np.max(np.abs(convnets.avgpool2_bwd(dy) - xt.grad.numpy())) < 1e-14


class _TorchR50H(torch.nn.Module):
    """Independent torch construction of the RGB-D encoder (normalise, avg-pool, ResNet50/2, compress)."""

    def __init__(self, p):
        super().__init__()
        self.p = p

    def forward(self, x):
        p = self.p
        mean = torch.tensor([0.485, 0.456, 0.406, 0.0], dtype=torch.float64).view(1, 4, 1, 1) * 255.0
        std = torch.tensor([0.229, 0.224, 0.225, 1.0 / 255.0], dtype=torch.float64).view(1, 4, 1, 1) * 255.0
        z = F.avg_pool2d((x - mean) / std, 2)

        def cg(z, c, g, s, pad, relu):
            z = F.conv2d(z, p[c + ".weight"], stride=s, padding=pad)
            z = F.group_norm(z, 16, p[g + ".weight"], p[g + ".bias"], eps=1e-5)
            return F.relu(z) if relu else z
        z = F.max_pool2d(cg(z, "enc.stem.conv", "enc.stem.gn", 2, 3, True), 3, 2, 1)
        cin = 32
        for li, (w, nb) in enumerate(zip(convnets.WIDTHS, convnets.R50_BLOCKS)):
            for bi in range(nb):
                s = 2 if (bi == 0 and li > 0) else 1
                pre = f"enc.layer{li + 1}.{bi}"
                a = cg(z, pre + ".conv1", pre + ".gn1", 1, 0, True)
                b = cg(a, pre + ".conv2", pre + ".gn2", s, 1, True)
                c3 = cg(b, pre + ".conv3", pre + ".gn3", 1, 0, False)
                sc = cg(z, pre + ".down.conv", pre + ".down.gn", s, 0, False) if (s != 1 or cin != 4 * w) else z
                z = F.relu(c3 + sc)
                cin = 4 * w
        return cg(z, "enc.compress.conv", "enc.compress.gn", 1, 1, True)


def test_resnet50h_matches_torch():
    lay = models.layout("rgbd")
    offs, P = models.offsets("rgbd")
    ent = [(offs[n][0], int(np.prod(s)), f) for n, s, f in lay]
    flat = synth.init_params(ent, P, 13).astype(np.float64)
    rng = np.random.default_rng(14)
    flat += rng.normal(0, 0.05, P)  # GN affine away from (1, 0)
    p = models.unpack("rgbd", flat)
    x = synth.rgbd_frames(rng, 1, 2, H=64, W=64)[0].astype(np.float64)  # [2][4][64][64] (smaller maps)
    feat, caches = convnets.resnet50h_fwd(x, p)
    pt = {k: _t(v, True) for k, v in p.items() if k.startswith("enc.")}
    xt = _t(x, True)
    ft = _TorchR50H(pt)(xt)
    assert feat.shape == tuple(ft.shape)
    assert np.max(np.abs(feat - ft.detach().numpy())) < 1e-10
    dz = rng.normal(size=feat.shape)
    (ft * _t(dz)).sum().backward()
    g = {}
    dx = convnets.resnet50h_bwd(dz, p, caches, g)
    assert np.max(np.abs(dx - xt.grad.numpy())) < 1e-9 * max(1.0, np.abs(xt.grad.numpy()).max())
    for k, v in pt.items():
        assert np.max(np.abs(g[k] - v.grad.numpy())) < 1e-9 * max(1.0, np.abs(v.grad.numpy()).max()), k


def test_rgbd_layout_size():
    # half-width ResNet50 (bottlenecks 3/4/6/3) + compression + FC 2048->512 + 2-layer LSTM-512 + head
    assert models.offsets("rgbd")[1] == 12459621


def test_rgbd_model_finite_differences():
    lay = models.layout("rgbd")
    offs, P = models.offsets("rgbd")
    ent = [(offs[n][0], int(np.prod(s)), f) for n, s, f in lay]
    flat = synth.init_params(ent, P, 15).astype(np.float64)
    ro = synth.rollout(1, 2, 16, obs_shape=(4, 256, 256), rnn_layers=2)
    batch = {k: ro[k][:, :2] for k in ("goal", "prev_action", "mask")}
    batch.update(obs=ro["obs"], h0=ro["h0"], c0=ro["c0"])
    lin = {k: v.astype(np.float64) if v.dtype != np.int32 else v for k, v in synth.random_loss_inputs(2, 17).items()}

    def loss(fl):
        lg, v, cache = models.forward("rgbd", fl, batch)
        st, dl, dv = ppo.loss_and_grad(lg.reshape(2, -1), v.reshape(-1), lin["actions"], lin["logp_old"],
                                       lin["values_old"], lin["returns"], lin["adv"], np.ones(2, bool))
        return st["total"], cache, dl.reshape(1, 2, -1), dv.reshape(1, 2)

    L, cache, dl, dv = loss(flat)
    g = models.backward("rgbd", flat, cache, dl, dv)
    rng = np.random.default_rng(18)
    for name in ["enc.stem.conv.weight", "enc.layer3.0.conv3.weight", "rnn.weight_hh_l0", "rnn.weight_ih_l1"]:
        o, s = offs[name]
        for i in rng.choice(int(np.prod(s)), 2, replace=False):
            fp, fm = flat.copy(), flat.copy()
            fp[o + i] += 1e-7
            fm[o + i] -= 1e-7
            fd = (loss(fp)[0] - loss(fm)[0]) / 2e-7
            assert abs(fd - g[o + i]) < 1e-4 * max(abs(fd), 1e-3), (name, i, fd, g[o + i])


# ---------------------------------------------------------------- SE-ResNeXt50/2 (NEXT-3, reading R9)
@pytest.mark.parametrize("C,O,groups,s", [(8, 8, 4, 1), (16, 32, 16, 2), (6, 9, 3, 1)])
def test_grouped_conv_matches_torch(C, O, groups, s):
    rng = np.random.default_rng(C + O)
    x = rng.normal(size=(2, C, 7, 7))
    W = rng.normal(size=(O, C // groups, 3, 3))
    y, cache = convnets.conv_fwd_grouped(x, W, s, 1, groups)
    xt, Wt = _t(x, True), _t(W, True)
    yt = F.conv2d(xt, Wt, stride=s, padding=1, groups=groups)
    assert np.max(np.abs(y - yt.detach().numpy())) < 1e-12
    dy = rng.normal(size=y.shape)
    (yt * _t(dy)).sum().backward()
    dx, dW = convnets.conv_bwd_grouped(dy, W, s, 1, cache)
    assert np.max(np.abs(dx - xt.grad.numpy())) < 1e-12 and np.max(np.abs(dW - Wt.grad.numpy())) < 1e-12
    # groups == 1 is the dense convolution
    yd, _ = convnets.conv_fwd_grouped(x, rng.normal(size=(O, C, 3, 3)), s, 1, 1)
    assert yd.shape[1] == O


def test_squeeze_excite_matches_torch():
    rng = np.random.default_rng(3)
    N, C, R = 3, 32, 4
    x = rng.normal(size=(N, C, 5, 6))
    W1, b1 = rng.normal(size=(R, C)) * 0.3, rng.normal(size=R) * 0.1
    W2, b2 = rng.normal(size=(C, R)) * 0.3, rng.normal(size=C) * 0.1
    y, cache = convnets.se_fwd(x, W1, b1, W2, b2)
    ts = [_t(a, True) for a in (x, W1, b1, W2, b2)]
    xt, W1t, b1t, W2t, b2t = ts
    st = torch.sigmoid(F.linear(F.relu(F.linear(xt.mean(dim=(2, 3)), W1t, b1t)), W2t, b2t))
    yt = xt * st[:, :, None, None]
    assert np.max(np.abs(y - yt.detach().numpy())) < 1e-14
    dy = rng.normal(size=y.shape)
    (yt * _t(dy)).sum().backward()
    got = convnets.se_bwd(dy, W1, W2, cache)
    for mine, ref in zip(got, ts):
        assert np.max(np.abs(mine - ref.grad.numpy())) < 1e-12
    # zero FC weights and biases: s = sigmoid(0) = 1/2 exactly (a pure channel halving)
    y0, _ = convnets.se_fwd(x, 0 * W1, 0 * b1, 0 * W2, 0 * b2)
    assert np.array_equal(y0, x * 0.5)


class _TorchSERX50H(torch.nn.Module):
    """Independent torch construction of the SE-ResNeXt50/2 RGB-D encoder (R9)."""

    def __init__(self, p):
        super().__init__()
        self.p = p

    def forward(self, x):
        p = self.p
        mean = torch.tensor([0.485, 0.456, 0.406, 0.0], dtype=torch.float64).view(1, 4, 1, 1) * 255.0
        std = torch.tensor([0.229, 0.224, 0.225, 1.0 / 255.0], dtype=torch.float64).view(1, 4, 1, 1) * 255.0
        z = F.avg_pool2d((x - mean) / std, 2)

        def cg(z, c, g, s, pad, relu, groups=1):
            z = F.conv2d(z, p[c + ".weight"], stride=s, padding=pad, groups=groups)
            z = F.group_norm(z, 16, p[g + ".weight"], p[g + ".bias"], eps=1e-5)
            return F.relu(z) if relu else z
        z = F.max_pool2d(cg(z, "enc.stem.conv", "enc.stem.gn", 2, 3, True), 3, 2, 1)
        cin = 32
        for li, (w, nb) in enumerate(zip(convnets.WIDTHS, convnets.R50_BLOCKS)):
            for bi in range(nb):
                s = 2 if (bi == 0 and li > 0) else 1
                pre = f"enc.layer{li + 1}.{bi}"
                a = cg(z, pre + ".conv1", pre + ".gn1", 1, 0, True)
                b = cg(a, pre + ".conv2", pre + ".gn2", s, 1, True, groups=16)
                c3 = cg(b, pre + ".conv3", pre + ".gn3", 1, 0, False)
                sq = torch.sigmoid(F.linear(F.relu(F.linear(c3.mean(dim=(2, 3)), p[pre + ".se.fc1.weight"],
                                                            p[pre + ".se.fc1.bias"])),
                                            p[pre + ".se.fc2.weight"], p[pre + ".se.fc2.bias"]))
                sc = cg(z, pre + ".down.conv", pre + ".down.gn", s, 0, False) if (s != 1 or cin != 4 * w) else z
                z = F.relu(c3 * sq[:, :, None, None] + sc)
                cin = 4 * w
        return cg(z, "enc.compress.conv", "enc.compress.gn", 1, 1, True)


def test_serx50h_matches_torch():
    lay = models.layout("serx50")
    offs, P = models.offsets("serx50")
    ent = [(offs[n][0], int(np.prod(s)), f) for n, s, f in lay]
    flat = synth.init_params(ent, P, 15).astype(np.float64)
    rng = np.random.default_rng(16)
    flat += rng.normal(0, 0.05, P)
    p = models.unpack("serx50", flat)
    x = synth.rgbd_frames(rng, 1, 2, H=64, W=64)[0].astype(np.float64)
    feat, caches = convnets.serx50h_fwd(x, p)
    pt = {k: _t(v, True) for k, v in p.items() if k.startswith("enc.")}
    xt = _t(x, True)
    ft = _TorchSERX50H(pt)(xt)
    assert feat.shape == tuple(ft.shape) == (2, 128, 1, 1)
    assert np.max(np.abs(feat - ft.detach().numpy())) < 1e-10
    dz = rng.normal(size=feat.shape)
    (ft * _t(dz)).sum().backward()
    g = {}
    dx = convnets.serx50h_bwd(dz, p, caches, g)
    assert np.max(np.abs(dx - xt.grad.numpy())) < 1e-9 * max(1.0, np.abs(xt.grad.numpy()).max())
    for k, v in pt.items():
        assert np.max(np.abs(g[k] - v.grad.numpy())) < 1e-9 * max(1.0, np.abs(v.grad.numpy()).max()), k


def test_serx50_layout():
    offs, P = models.offsets("serx50")
    assert offs["enc.layer1.0.conv2.weight"][1] == (64, 4, 3, 3)      # 16 groups of 4 channels
    assert offs["enc.layer4.2.conv2.weight"][1] == (512, 32, 3, 3)
    assert offs["enc.layer4.2.se.fc1.weight"][1] == (64, 1024) and offs["enc.layer1.0.se.fc2.bias"][1] == (128,)
    assert P == 13321789
