"""Visual-encoder layers with manual backward passes (Depth / RGB-D agents, steps a5/a7).

Test infrastructure only.  NumPy float64, NCHW, textbook definitions:
  * Conv2d without bias (ResNet convention; every conv is followed by GroupNorm),
    computed as im2col + matmul: y[n,o,i,j] = sum_{c,u,v} W[o,c,u,v] x[n,c,i*s-p+u,j*s-p+v];
  * GroupNorm ("replace every BatchNorm layer with GroupNorm"; reading Z19:
    G = 16 groups, eps = 1e-5, per-channel affine): biased variance over (C/G, H, W) per sample;
  * ReLU; MaxPool 3x3 / stride 2 / pad 1 (Z23) with the first maximum in (u, v) scan order
    taking the gradient;
  * half-width ResNet18 ("number of output channels at every layer reduced by half",
    reading Z23: stem 7x7/2 + maxpool, BasicBlocks 32/64/128/256, stride on the first block of
    layers 2-4 with a 1x1/stride conv + GN shortcut), then the 3x3 compression conv to 128
    channels + GN + ReLU (Z20);
  * half-width ResNet50 for the RGB-D agent (bottlenecks [3, 4, 6, 3], 2x2 average pooling of the
    256^2 input first, channel-wise RGB normalisation P:L367) -> 1024x4x4 -> compression to 128x4x4;
  * half-width SE-ResNeXt50 (NEXT-3; reading R9 in DESIGN.md): the ResNet50/2
    topology with each bottleneck's 3x3 convolution grouped (cardinality 16 over an inner width of
    2 x planes, Xie et al.'s aggregated transformations) and a squeeze-excitation module (Hu et al.:
    global average pool -> FC C/16 + ReLU -> FC C + sigmoid -> channel scale; reduction 16) on the
    residual branch before the addition.
"""
import numpy as np


def _pad(x, p):
    return np.pad(x, ((0, 0), (0, 0), (p, p), (p, p))) if p else x


def im2col(x, kh, kw, s, p):
    """x [N][C][H][W] -> cols [N*Ho*Wo][C*kh*kw] (column index c*kh*kw + u*kw + v), Ho, Wo."""
    N, C, H, W = x.shape
    xp = _pad(x, p)
    Ho = (H + 2 * p - kh) // s + 1
    Wo = (W + 2 * p - kw) // s + 1
    cols = np.empty((N, Ho, Wo, C, kh, kw))
    for u in range(kh):
        for v in range(kw):
            cols[:, :, :, :, u, v] = xp[:, :, u:u + s * Ho:s, v:v + s * Wo:s].transpose(0, 2, 3, 1)
    return cols.reshape(N * Ho * Wo, C * kh * kw), Ho, Wo


def col2im(cols, shape, kh, kw, s, p, Ho, Wo):
    N, C, H, W = shape
    xp = np.zeros((N, C, H + 2 * p, W + 2 * p))
    c6 = cols.reshape(N, Ho, Wo, C, kh, kw)
    for u in range(kh):
        for v in range(kw):
            xp[:, :, u:u + s * Ho:s, v:v + s * Wo:s] += c6[:, :, :, :, u, v].transpose(0, 3, 1, 2)
    return xp[:, :, p:p + H, p:p + W] if p else xp


def conv_fwd(x, W, s, p):
    N = x.shape[0]
    O, C, kh, kw = W.shape
    cols, Ho, Wo = im2col(x, kh, kw, s, p)
    y = cols @ W.reshape(O, -1).T
    return y.reshape(N, Ho, Wo, O).transpose(0, 3, 1, 2), (x.shape, cols, Ho, Wo)


def conv_bwd(dy, W, s, p, cache):
    shape, cols, Ho, Wo = cache
    O, C, kh, kw = W.shape
    d2 = dy.transpose(0, 2, 3, 1).reshape(-1, O)
    dW = (d2.T @ cols).reshape(W.shape)
    dx = col2im(d2 @ W.reshape(O, -1), shape, kh, kw, s, p, Ho, Wo)
    return dx, dW


def gn_fwd(x, gamma, beta, G=16, eps=1e-5):
    N, C, H, W = x.shape
    xg = x.reshape(N, G, -1)
    mu = xg.mean(axis=2, keepdims=True)
    var = ((xg - mu) ** 2).mean(axis=2, keepdims=True)
    rstd = 1.0 / np.sqrt(var + eps)
    xhat = ((xg - mu) * rstd).reshape(N, C, H, W)
    return xhat * gamma[None, :, None, None] + beta[None, :, None, None], (xhat, rstd, G)


def gn_bwd(dy, gamma, cache):
    xhat, rstd, G = cache
    N, C, H, W = dy.shape
    dgamma = (dy * xhat).sum(axis=(0, 2, 3))
    dbeta = dy.sum(axis=(0, 2, 3))
    dxhat = (dy * gamma[None, :, None, None]).reshape(N, G, -1)
    xh = xhat.reshape(N, G, -1)
    m = dxhat.shape[2]
    dx = rstd * (dxhat - dxhat.mean(axis=2, keepdims=True) - xh * (dxhat * xh).mean(axis=2, keepdims=True))
    return dx.reshape(N, C, H, W), dgamma, dbeta


def maxpool_fwd(x, k=3, s=2, p=1):
    N, C, H, W = x.shape
    xp = np.pad(x, ((0, 0), (0, 0), (p, p), (p, p)), constant_values=-np.inf)
    Ho = (H + 2 * p - k) // s + 1
    Wo = (W + 2 * p - k) // s + 1
    win = np.stack([xp[:, :, u:u + s * Ho:s, v:v + s * Wo:s] for u in range(k) for v in range(k)], axis=-1)
    arg = win.argmax(axis=-1)  # first maximum in (u, v) scan order
    return win.max(axis=-1), (x.shape, arg, k, s, p, Ho, Wo)


def maxpool_bwd(dy, cache):
    shape, arg, k, s, p, Ho, Wo = cache
    N, C, H, W = shape
    dxp = np.zeros((N, C, H + 2 * p, W + 2 * p))
    for u in range(k):
        for v in range(k):
            sel = (arg == u * k + v)
            dxp[:, :, u:u + s * Ho:s, v:v + s * Wo:s] += np.where(sel, dy, 0.0)
    return dxp[:, :, p:p + H, p:p + W]


# ---------------------------------------------------------------- half-width ResNet18
WIDTHS = (32, 64, 128, 256)


def resnet18h_spec(in_ch):
    """Ordered (name, kind, shape, stride, pad) of the encoder's parameter tensors."""
    spec = [("enc.stem.conv", "conv", (32, in_ch, 7, 7), 2, 3), ("enc.stem.gn", "gn", (32,), 0, 0)]
    cin = 32
    for li, c in enumerate(WIDTHS):
        for bi in range(2):
            s = 2 if (bi == 0 and li > 0) else 1
            pre = f"enc.layer{li + 1}.{bi}"
            spec += [(pre + ".conv1", "conv", (c, cin, 3, 3), s, 1), (pre + ".gn1", "gn", (c,), 0, 0),
                     (pre + ".conv2", "conv", (c, c, 3, 3), 1, 1), (pre + ".gn2", "gn", (c,), 0, 0)]
            if s != 1 or cin != c:
                spec += [(pre + ".down.conv", "conv", (c, cin, 1, 1), s, 0), (pre + ".down.gn", "gn", (c,), 0, 0)]
            cin = c
    spec += [("enc.compress.conv", "conv", (128, 256, 3, 3), 1, 1), ("enc.compress.gn", "gn", (128,), 0, 0)]
    return spec


def _conv_gn(x, p, cname, gname, s, pad, relu, caches):
    y, cc = conv_fwd(x, p[cname + ".weight"], s, pad)
    z, gc = gn_fwd(y, p[gname + ".weight"], p[gname + ".bias"])
    caches[cname] = (cc, gc, s, pad)
    if relu:
        caches[cname + ".relu"] = z > 0
        z = np.maximum(z, 0.0)
    return z


def _conv_gn_bwd(dz, p, cname, gname, relu, caches, g):
    cc, gc, s, pad = caches[cname]
    if relu:
        dz = dz * caches[cname + ".relu"]
    dy, g[gname + ".weight"], g[gname + ".bias"] = gn_bwd(dz, p[gname + ".weight"], gc)
    dx, g[cname + ".weight"] = conv_bwd(dy, p[cname + ".weight"], s, pad, cc)
    return dx


def resnet18h_fwd(x, p):
    """x [N][C][64][64] (or larger) -> feature [N][128][h][w] (after compression conv + GN + ReLU)."""
    caches = {}
    z = _conv_gn(x, p, "enc.stem.conv", "enc.stem.gn", 2, 3, True, caches)
    z, caches["pool"] = maxpool_fwd(z)
    cin = 32
    for li, c in enumerate(WIDTHS):
        for bi in range(2):
            s = 2 if (bi == 0 and li > 0) else 1
            pre = f"enc.layer{li + 1}.{bi}"
            a = _conv_gn(z, p, pre + ".conv1", pre + ".gn1", s, 1, True, caches)
            b = _conv_gn(a, p, pre + ".conv2", pre + ".gn2", 1, 1, False, caches)
            sc = z
            if s != 1 or cin != c:
                sc = _conv_gn(z, p, pre + ".down.conv", pre + ".down.gn", s, 0, False, caches)
            out = b + sc
            caches[pre + ".out"] = out > 0
            z = np.maximum(out, 0.0)
            cin = c
    z = _conv_gn(z, p, "enc.compress.conv", "enc.compress.gn", 1, 1, True, caches)
    return z, caches


def resnet18h_bwd(dz, p, caches, g):
    dz = _conv_gn_bwd(dz, p, "enc.compress.conv", "enc.compress.gn", True, caches, g)
    blocks = [(li, bi) for li in range(4) for bi in range(2)]
    for li, bi in reversed(blocks):
        c = WIDTHS[li]
        cin = (32 if li == 0 else WIDTHS[li - 1]) if bi == 0 else c
        s = 2 if (bi == 0 and li > 0) else 1
        pre = f"enc.layer{li + 1}.{bi}"
        dout = dz * caches[pre + ".out"]
        da = _conv_gn_bwd(dout, p, pre + ".conv2", pre + ".gn2", False, caches, g)
        dx = _conv_gn_bwd(da, p, pre + ".conv1", pre + ".gn1", True, caches, g)
        if s != 1 or cin != c:
            dx = dx + _conv_gn_bwd(dout, p, pre + ".down.conv", pre + ".down.gn", False, caches, g)
        else:
            dx = dx + dout
        dz = dx
    dz = maxpool_bwd(dz, caches["pool"])
    dx = _conv_gn_bwd(dz, p, "enc.stem.conv", "enc.stem.gn", True, caches, g)
    return dx


# ---------------------------------------------------------------- RGB-D agent (configs[3])
# P:L212 / P:L582 (half-width ResNet50 "1024x4x4"), reading Z23: 2x2 average pooling of the 256^2
# input, stem 7x7/2 conv + GN + ReLU + 3x3/2 max-pool, bottleneck blocks [3, 4, 6, 3] with widths
# 32/64/128/256 (outputs x4), stride on the 3x3 (v1.5) of the first block of layers 2-4, 1x1/stride
# conv + GN shortcut when the shape changes; compression 3x3 conv 1024 -> 128 + GN + ReLU (Z20).
# RGB channels are normalised channel-wise before the encoder (reading R7).
R50_BLOCKS = (3, 4, 6, 3)
RGB_MEAN = (0.485 * 255.0, 0.456 * 255.0, 0.406 * 255.0)
RGB_STD = (0.229 * 255.0, 0.224 * 255.0, 0.225 * 255.0)


def avgpool2_fwd(x):
    """2x2 / stride 2 average pooling (H, W even)."""
    N, C, H, W = x.shape
    return x.reshape(N, C, H // 2, 2, W // 2, 2).mean(axis=(3, 5))


def avgpool2_bwd(dy):
    return np.repeat(np.repeat(dy, 2, axis=2), 2, axis=3) / 4.0


def rgbd_normalize(x):
    """x [N][4][H][W]: RGB in [0, 255] -> (x - mean_c) / std_c; depth (channel 3) unchanged."""
    out = np.array(x, dtype=np.float64, copy=True)
    for c in range(3):
        out[:, c] = (out[:, c] - RGB_MEAN[c]) / RGB_STD[c]
    return out


def resnet50h_spec(in_ch):
    """Ordered (name, kind, shape, stride, pad) of the RGB-D encoder's parameter tensors."""
    spec = [("enc.stem.conv", "conv", (32, in_ch, 7, 7), 2, 3), ("enc.stem.gn", "gn", (32,), 0, 0)]
    cin = 32
    for li, (w, nb) in enumerate(zip(WIDTHS, R50_BLOCKS)):
        for bi in range(nb):
            s = 2 if (bi == 0 and li > 0) else 1
            pre = f"enc.layer{li + 1}.{bi}"
            spec += [(pre + ".conv1", "conv", (w, cin, 1, 1), 1, 0), (pre + ".gn1", "gn", (w,), 0, 0),
                     (pre + ".conv2", "conv", (w, w, 3, 3), s, 1), (pre + ".gn2", "gn", (w,), 0, 0),
                     (pre + ".conv3", "conv", (4 * w, w, 1, 1), 1, 0), (pre + ".gn3", "gn", (4 * w,), 0, 0)]
            if s != 1 or cin != 4 * w:
                spec += [(pre + ".down.conv", "conv", (4 * w, cin, 1, 1), s, 0),
                         (pre + ".down.gn", "gn", (4 * w,), 0, 0)]
            cin = 4 * w
    spec += [("enc.compress.conv", "conv", (128, 1024, 3, 3), 1, 1), ("enc.compress.gn", "gn", (128,), 0, 0)]
    return spec


def resnet50h_fwd(x, p):
    """x [N][4][256][256] (raw RGB-D) -> feature [N][128][4][4]."""
    caches = {}
    z = avgpool2_fwd(rgbd_normalize(x))
    z = _conv_gn(z, p, "enc.stem.conv", "enc.stem.gn", 2, 3, True, caches)
    z, caches["pool"] = maxpool_fwd(z)
    cin = 32
    for li, (w, nb) in enumerate(zip(WIDTHS, R50_BLOCKS)):
        for bi in range(nb):
            s = 2 if (bi == 0 and li > 0) else 1
            pre = f"enc.layer{li + 1}.{bi}"
            a = _conv_gn(z, p, pre + ".conv1", pre + ".gn1", 1, 0, True, caches)
            b = _conv_gn(a, p, pre + ".conv2", pre + ".gn2", s, 1, True, caches)
            c3 = _conv_gn(b, p, pre + ".conv3", pre + ".gn3", 1, 0, False, caches)
            sc = z
            if s != 1 or cin != 4 * w:
                sc = _conv_gn(z, p, pre + ".down.conv", pre + ".down.gn", s, 0, False, caches)
            out = c3 + sc
            caches[pre + ".out"] = out > 0
            z = np.maximum(out, 0.0)
            cin = 4 * w
    z = _conv_gn(z, p, "enc.compress.conv", "enc.compress.gn", 1, 1, True, caches)
    return z, caches


def resnet50h_bwd(dz, p, caches, g):
    """Parameter gradients into g; returns the gradient wrt the raw input."""
    dz = _conv_gn_bwd(dz, p, "enc.compress.conv", "enc.compress.gn", True, caches, g)
    blocks = []
    cin = 32
    for li, (w, nb) in enumerate(zip(WIDTHS, R50_BLOCKS)):
        for bi in range(nb):
            blocks.append((li, bi, w, cin))
            cin = 4 * w
    for li, bi, w, cin in reversed(blocks):
        s = 2 if (bi == 0 and li > 0) else 1
        pre = f"enc.layer{li + 1}.{bi}"
        dout = dz * caches[pre + ".out"]
        db = _conv_gn_bwd(dout, p, pre + ".conv3", pre + ".gn3", False, caches, g)
        da = _conv_gn_bwd(db, p, pre + ".conv2", pre + ".gn2", True, caches, g)
        dx = _conv_gn_bwd(da, p, pre + ".conv1", pre + ".gn1", True, caches, g)
        if s != 1 or cin != 4 * w:
            dx = dx + _conv_gn_bwd(dout, p, pre + ".down.conv", pre + ".down.gn", False, caches, g)
        else:
            dx = dx + dout
        dz = dx
    dz = maxpool_bwd(dz, caches["pool"])
    dz = _conv_gn_bwd(dz, p, "enc.stem.conv", "enc.stem.gn", True, caches, g)
    dx = avgpool2_bwd(dz)
    for c in range(3):
        dx[:, c] /= RGB_STD[c]
    return dx


# ---------------------------------------------------------------- SE-ResNeXt50/2 (NEXT-3)
SERX_CARD = 16   # cardinality of the grouped 3x3 convolutions (R9)
R101_BLOCKS = (3, 4, 23, 3)  # SE-ResNeXt101 ("SE-ResNeXt101 + 1024-d LSTM")
SE_RED = 16      # squeeze-excitation reduction


def conv_fwd_grouped(x, W, s, p, groups):
    """Grouped convolution: input and output channels split into `groups` equal parts, group g's
    outputs see only group g's inputs; W [O][C/groups][k][k]."""
    C, O = x.shape[1], W.shape[0]
    cg, og = C // groups, O // groups
    ys, cs = [], []
    for g in range(groups):
        y, cc = conv_fwd(x[:, g * cg:(g + 1) * cg], W[g * og:(g + 1) * og], s, p)
        ys.append(y)
        cs.append(cc)
    return np.concatenate(ys, axis=1), (cs, groups)


def conv_bwd_grouped(dy, W, s, p, cache):
    cs, groups = cache
    O = W.shape[0]
    og = O // groups
    dxs, dWs = [], []
    for g in range(groups):
        dx, dW = conv_bwd(dy[:, g * og:(g + 1) * og], W[g * og:(g + 1) * og], s, p, cs[g])
        dxs.append(dx)
        dWs.append(dW)
    return np.concatenate(dxs, axis=1), np.concatenate(dWs, axis=0)


def sigmoid(x):
    return 1.0 / (1.0 + np.exp(-x))


def se_fwd(x, W1, b1, W2, b2):
    """y = x * s[:, :, None, None], s = sigmoid(W2 relu(W1 mean_hw(x) + b1) + b2)."""
    pooled = x.mean(axis=(2, 3))
    a1 = pooled @ W1.T + b1
    h = np.maximum(a1, 0.0)
    sc = sigmoid(h @ W2.T + b2)
    return x * sc[:, :, None, None], (x, pooled, a1, h, sc)


def se_bwd(dy, W1, W2, cache):
    x, pooled, a1, h, sc = cache
    HW = x.shape[2] * x.shape[3]
    ds = (dy * x).sum(axis=(2, 3))
    da2 = ds * sc * (1.0 - sc)
    dW2, db2 = da2.T @ h, da2.sum(0)
    da1 = (da2 @ W2) * (a1 > 0)
    dW1, db1 = da1.T @ pooled, da1.sum(0)
    dpooled = da1 @ W1
    dx = dy * sc[:, :, None, None] + dpooled[:, :, None, None] / HW
    return dx, dW1, db1, dW2, db2


def serx50h_spec(in_ch, blocks=R50_BLOCKS):
    """Ordered (name, kind, shape, stride, pad) of the SE-ResNeXt50/2 (blocks R101_BLOCKS: 101/2) encoder's
    parameter tensors (kind "gconv": grouped, cardinality SERX_CARD; "fc": SE linear layers with a bias)."""
    spec = [("enc.stem.conv", "conv", (32, in_ch, 7, 7), 2, 3), ("enc.stem.gn", "gn", (32,), 0, 0)]
    cin = 32
    for li, (w, nb) in enumerate(zip(WIDTHS, blocks)):
        for bi in range(nb):
            s = 2 if (bi == 0 and li > 0) else 1
            pre = f"enc.layer{li + 1}.{bi}"
            wi, co = 2 * w, 4 * w
            spec += [(pre + ".conv1", "conv", (wi, cin, 1, 1), 1, 0), (pre + ".gn1", "gn", (wi,), 0, 0),
                     (pre + ".conv2", "gconv", (wi, wi // SERX_CARD, 3, 3), s, 1), (pre + ".gn2", "gn", (wi,), 0, 0),
                     (pre + ".conv3", "conv", (co, wi, 1, 1), 1, 0), (pre + ".gn3", "gn", (co,), 0, 0),
                     (pre + ".se.fc1", "fc", (co // SE_RED, co), 0, 0), (pre + ".se.fc2", "fc", (co, co // SE_RED), 0, 0)]
            if s != 1 or cin != co:
                spec += [(pre + ".down.conv", "conv", (co, cin, 1, 1), s, 0),
                         (pre + ".down.gn", "gn", (co,), 0, 0)]
            cin = co
    spec += [("enc.compress.conv", "conv", (128, 1024, 3, 3), 1, 1), ("enc.compress.gn", "gn", (128,), 0, 0)]
    return spec


def serx50h_fwd(x, p, blocks=R50_BLOCKS):
    """x [N][4][256][256] (raw RGB-D) -> feature [N][128][4][4]."""
    caches = {}
    z = avgpool2_fwd(rgbd_normalize(x))
    z = _conv_gn(z, p, "enc.stem.conv", "enc.stem.gn", 2, 3, True, caches)
    z, caches["pool"] = maxpool_fwd(z)
    cin = 32
    for li, (w, nb) in enumerate(zip(WIDTHS, blocks)):
        for bi in range(nb):
            s = 2 if (bi == 0 and li > 0) else 1
            pre = f"enc.layer{li + 1}.{bi}"
            a = _conv_gn(z, p, pre + ".conv1", pre + ".gn1", 1, 0, True, caches)
            y2, cc2 = conv_fwd_grouped(a, p[pre + ".conv2.weight"], s, 1, SERX_CARD)
            b, gc2 = gn_fwd(y2, p[pre + ".gn2.weight"], p[pre + ".gn2.bias"])
            caches[pre + ".conv2"] = (cc2, gc2, s, 1)
            caches[pre + ".conv2.relu"] = b > 0
            b = np.maximum(b, 0.0)
            c3 = _conv_gn(b, p, pre + ".conv3", pre + ".gn3", 1, 0, False, caches)
            e, caches[pre + ".se"] = se_fwd(c3, p[pre + ".se.fc1.weight"], p[pre + ".se.fc1.bias"],
                                            p[pre + ".se.fc2.weight"], p[pre + ".se.fc2.bias"])
            sc = z
            if s != 1 or cin != 4 * w:
                sc = _conv_gn(z, p, pre + ".down.conv", pre + ".down.gn", s, 0, False, caches)
            out = e + sc
            caches[pre + ".out"] = out > 0
            z = np.maximum(out, 0.0)
            cin = 4 * w
    z = _conv_gn(z, p, "enc.compress.conv", "enc.compress.gn", 1, 1, True, caches)
    return z, caches


def serx50h_bwd(dz, p, caches, g, blocks_per_layer=R50_BLOCKS):
    """Parameter gradients into g; returns the gradient wrt the raw input."""
    dz = _conv_gn_bwd(dz, p, "enc.compress.conv", "enc.compress.gn", True, caches, g)
    blocks = []
    cin = 32
    for li, (w, nb) in enumerate(zip(WIDTHS, blocks_per_layer)):
        for bi in range(nb):
            blocks.append((li, bi, w, cin))
            cin = 4 * w
    for li, bi, w, cin in reversed(blocks):
        s = 2 if (bi == 0 and li > 0) else 1
        pre = f"enc.layer{li + 1}.{bi}"
        dout = dz * caches[pre + ".out"]
        de, g[pre + ".se.fc1.weight"], g[pre + ".se.fc1.bias"], g[pre + ".se.fc2.weight"], g[pre + ".se.fc2.bias"] = \
            se_bwd(dout, p[pre + ".se.fc1.weight"], p[pre + ".se.fc2.weight"], caches[pre + ".se"])
        db = _conv_gn_bwd(de, p, pre + ".conv3", pre + ".gn3", False, caches, g)
        cc2, gc2, s2, pad2 = caches[pre + ".conv2"]
        db = db * caches[pre + ".conv2.relu"]
        dy2, g[pre + ".gn2.weight"], g[pre + ".gn2.bias"] = gn_bwd(db, p[pre + ".gn2.weight"], gc2)
        da, g[pre + ".conv2.weight"] = conv_bwd_grouped(dy2, p[pre + ".conv2.weight"], s2, pad2, cc2)
        dx = _conv_gn_bwd(da, p, pre + ".conv1", pre + ".gn1", True, caches, g)
        if s != 1 or cin != 4 * w:
            dx = dx + _conv_gn_bwd(dout, p, pre + ".down.conv", pre + ".down.gn", False, caches, g)
        else:
            dx = dx + dout
        dz = dx
    dz = maxpool_bwd(dz, caches["pool"])
    dz = _conv_gn_bwd(dz, p, "enc.stem.conv", "enc.stem.gn", True, caches, g)
    dx = avgpool2_bwd(dz)
    for c in range(3):
        dx[:, c] /= RGB_STD[c]
    return dx
