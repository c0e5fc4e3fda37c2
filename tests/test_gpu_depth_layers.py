"""Layer-level parity of the Depth encoder (configs[2]) through its diagnostic C entries, against
oracle.convnets (fp64, NCHW; transposed to the kernels' NHWC here).

Tolerances:
  conv forward (bf16 hi/lo operand planes, the stem's warp MMAs too; the SIMT stem in fp32): |err| <= 2e-5 * (|x| conv |W|);
  conv dgrad / wgrad (bf16 operands, fp32 accumulation): |err| <= 1e-2 * the same op on |.|;
  GroupNorm (fp32 SIMT): 1e-4 relative to the tensor's scale (its input gradient is delivered in
  bf16: + 2^-8 relative); max-pool: exact forward."""
import numpy as np
import pytest
import torch

from oracle import convnets

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def dd():
    if not torch.cuda.is_available():
        pytest.skip("needs a GPU")
    import paper_1911_00357_b200 as m
    return m


@pytest.fixture(scope="module")
def ctx(dd):
    c = dd.Context(0, 1)
    yield c
    c.close()


def cu(a):
    return torch.from_numpy(np.ascontiguousarray(a, dtype=np.float32)).cuda()


def nhwc(a):
    return np.ascontiguousarray(a.transpose(0, 2, 3, 1))


def nchw(a):
    return np.ascontiguousarray(a.transpose(0, 3, 1, 2))


@pytest.mark.parametrize("F,H,Ci,Co,k,s,p", [
    (3, 64, 1, 32, 7, 2, 3),    # stem
    (2, 16, 32, 32, 3, 1, 1),   # layer1
    (2, 16, 32, 64, 3, 2, 1),   # layer2.0.conv1
    (2, 16, 32, 64, 1, 2, 0),   # layer2.0.down
    (5, 2, 256, 128, 3, 1, 1),  # compress (2x2 maps)
    (3, 7, 24, 40, 3, 2, 1),    # ragged
    (4, 5, 8, 16, 1, 1, 0),     # 1x1 / stride 1
    (2, 9, 1, 16, 3, 1, 1),     # single-channel (SIMT stem kernels: 81 pixels, not a multiple of 16)
    (2, 16, 1, 16, 5, 1, 2),    # single-channel, warp-MMA stem at another geometry (Co 16, 5x5 s1)
    (3, 24, 1, 32, 3, 2, 1),    # single-channel, warp-MMA stem (3x3 s2, 144 pixels)
    (2, 32, 8, 32, 7, 2, 3),    # RGB-D stem (4 channels padded to 8)
    (2, 8, 64, 256, 1, 1, 0),   # bottleneck 1x1 expansion
    (2, 4, 1024, 128, 3, 1, 1),   # RGB-D compression (1024 -> 128 at 4x4)
    (256, 16, 32, 32, 3, 1, 1),   # layer1 at the config's minibatch (F = 256 frames: 512 tiles)
    (256, 2, 256, 256, 3, 1, 1),  # layer4 at the config's minibatch (split-K)
    (7, 9, 96, 40, 3, 1, 1)])     # odd spatial size, 3 channel slices, ragged M
@pytest.mark.parametrize("engine", ["tma", "cpasync"])
def test_conv2d(dd, ctx, F, H, Ci, Co, k, s, p, engine):
    dd.ddppo_set_conv_engine(ctx, engine)
    rng = np.random.default_rng(F * 100 + H + Ci + Co + k)
    x = rng.normal(size=(F, Ci, H, H)).astype(np.float32)
    x[x < -0.5] = 0.0  # post-ReLU-like inputs with exact zeros
    W = (rng.normal(size=(Co, Ci, k, k)) / np.sqrt(Ci * k * k)).astype(np.float32)
    y_o, cache = convnets.conv_fwd(x.astype(np.float64), W.astype(np.float64), s, p)
    Ho = y_o.shape[2]
    dy = rng.normal(size=y_o.shape).astype(np.float32)
    dx_o, dW_o = convnets.conv_bwd(dy.astype(np.float64), W.astype(np.float64), s, p, cache)
    # magnitudes for the error bounds: the same ops on absolute values
    ya, ca = convnets.conv_fwd(np.abs(x).astype(np.float64), np.abs(W).astype(np.float64), s, p)
    dxa, dWa = convnets.conv_bwd(np.abs(dy).astype(np.float64), np.abs(W).astype(np.float64), s, p, ca)

    y = torch.zeros((F, Ho, Ho, Co), device="cuda")
    dx = torch.full((F, H, H, Ci), 7.0, device="cuda")
    dW = torch.full((Co, Ci, k, k), 7.0, device="cuda")
    keep = dd.ddppo_debug_conv2d(ctx, cu(nhwc(x)), cu(W), F, H, H, Ci, Co, k, s, p, y=y, dy=cu(nhwc(dy)), dx=dx,
                                 dw=dW)
    torch.cuda.synchronize()
    del keep
    ctx.check()
    assert np.all(np.abs(nchw(y.cpu().numpy()) - y_o) <= 2e-5 * ya + 1e-7)
    if Ci > 1:  # the stem (1 input channel) has no input gradient
        assert np.all(np.abs(nchw(dx.cpu().numpy()) - dx_o) <= 1e-2 * dxa + 1e-6)
    assert np.all(np.abs(dW.cpu().numpy() - dW_o) <= 1e-2 * dWa + 1e-6)


@pytest.mark.parametrize("F,HW,C,relu,res", [(3, 1024, 32, True, False), (2, 64, 64, False, True),
                                             (5, 4, 256, True, True), (4, 4, 128, True, False),
                                             (2, 9, 16, False, False), (2, 16, 1024, True, True),
                                             (2, 256, 512, False, False)])
def test_groupnorm(dd, ctx, F, HW, C, relu, res):
    rng = np.random.default_rng(F + HW + C)
    y = (rng.normal(size=(F, C, HW, 1)) * 2 + 0.5).astype(np.float32)
    gamma = rng.normal(1.0, 0.3, C).astype(np.float32)
    beta = rng.normal(0.0, 0.3, C).astype(np.float32)
    r = rng.normal(size=y.shape).astype(np.float32) if res else np.zeros_like(y)
    z_o, gc = convnets.gn_fwd(y.astype(np.float64), gamma.astype(np.float64), beta.astype(np.float64))
    z_o = z_o + r
    if relu:
        mask = z_o > 0
        z_o = np.maximum(z_o, 0)
    dz = rng.normal(size=y.shape).astype(np.float32)
    dzm = dz * mask if relu else dz.astype(np.float64)
    dy_o, dg_o, db_o = convnets.gn_bwd(dzm, gamma.astype(np.float64), gc)

    z = torch.zeros((F, HW, C), device="cuda")
    stats = torch.zeros((F, 16, 2), device="cuda")
    dy = torch.zeros((F, HW, C), device="cuda")
    dg = torch.zeros(C, device="cuda")
    db = torch.zeros(C, device="cuda")
    keep = dd.ddppo_debug_groupnorm(ctx, cu(nhwc(y)), cu(gamma), cu(beta), F, HW, C, relu, z, stats,
                                    residual=cu(nhwc(r)) if res else None, dz=cu(nhwc(dz)), dy=dy, dgamma=dg,
                                    dbeta=db)
    torch.cuda.synchronize()
    del keep
    zz = nchw(z.cpu().numpy().reshape(F, HW, 1, C))
    assert np.max(np.abs(zz - z_o)) <= 1e-4 * np.abs(z_o).max()
    dyy = nchw(dy.cpu().numpy().reshape(F, HW, 1, C))
    # dy is delivered rounded to bf16 (the gradient GEMMs' operand format): 2^-8 relative
    assert np.all(np.abs(dyy - dy_o) <= 2.0 ** -8 * np.abs(dy_o) + 1e-4 * np.abs(dy_o).max())
    assert np.max(np.abs(dg.cpu().numpy() - dg_o)) <= 1e-4 * np.abs(dg_o).max()
    assert np.max(np.abs(db.cpu().numpy() - db_o)) <= 1e-4 * np.abs(db_o).max()


@pytest.mark.parametrize("F,H,C", [(3, 32, 32), (2, 7, 12), (1, 2, 16), (2, 9, 4), (2, 10, 8)])  # even H: 2x2-block backward
def test_maxpool(dd, ctx, F, H, C):
    rng = np.random.default_rng(F * H * C)
    x = np.maximum(rng.normal(size=(F, C, H, H)), 0).astype(np.float32)  # ReLU zeros: ties
    y_o, cache = convnets.maxpool_fwd(x.astype(np.float64))
    dy = rng.normal(size=y_o.shape).astype(np.float32)
    dx_o = convnets.maxpool_bwd(dy.astype(np.float64), cache)
    Ho = y_o.shape[2]
    y = torch.zeros((F, Ho, Ho, C), device="cuda")
    arg = torch.zeros((F, Ho, Ho, C), dtype=torch.uint8, device="cuda")
    dx = torch.zeros((F, H, H, C), device="cuda")
    dd.ddppo_debug_maxpool(ctx, cu(nhwc(x)), F, H, H, C, y, arg, dy=cu(nhwc(dy)), dx=dx)
    torch.cuda.synchronize()
    assert np.array_equal(nchw(y.cpu().numpy()), y_o.astype(np.float32))
    assert np.array_equal(nchw(arg.cpu().numpy()), cache[1])  # the first maximum (torch's tie rule)
    assert np.max(np.abs(nchw(dx.cpu().numpy()) - dx_o)) <= 1e-6
