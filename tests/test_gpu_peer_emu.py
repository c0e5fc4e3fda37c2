"""The NVLink peer-memory exchange kernels (a8 v1 all-read, a8 v2 reduce-scatter -> shard Adam ->
all-gather, a10 counts) on ONE GPU: N in {2, 4, 8} ranks emulated over N buffer sets by
ddppo_debug_peer_a8 / ddppo_debug_peer_counts, which run exactly the multi-GPU kernels (flag
barrier, rank-ordered sums, shard norm partials, staged shards).

Bars: the gradient sum is bit-exact against an fp32 rank-ordered sum (K16 v2 "sums
in fixed rank order in fp32"); parameters are bit-identical on every emulated rank; the update
matches the oracle's Eq. 3 + clip + Adam (oracle/optim.py, fp64) within 1e-4 relative; counts are
exact int64 sums."""
import numpy as np
import pytest
import torch

import paper_1911_00357_b200 as dd
from oracle import optim

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def ctx():
    c = dd.Context(0, 1, device=0)
    yield c
    c.close()


def _shard(P, N, r):
    Q = P // 4
    lo, hi = Q * r // N * 4, Q * (r + 1) // N * 4
    return lo, (P if r == N - 1 else hi)


@pytest.mark.parametrize("mode", ["allread", "sharded"])
@pytest.mark.parametrize("N,P,step", [(2, 890661, 1), (4, 4099, 3), (8, 5588741, 1), (8, 37, 2), (3, 1000003, 5)])
def test_peer_a8_emulated(ctx, mode, N, P, step):
    g = torch.Generator().manual_seed(N * 1000 + P % 997 + step)
    grads = [torch.randn(P, generator=g) * (0.02 * (r + 1)) for r in range(N)]
    p0 = torch.randn(P, generator=g) * 0.05
    m0 = torch.randn(P, generator=g) * 1e-3 if step > 1 else torch.zeros(P)
    v0 = torch.rand(P, generator=g) * 1e-5 if step > 1 else torch.zeros(P)
    dev = lambda t: t.clone().cuda()  # noqa: E731
    gd = [dev(x) for x in grads]
    pr, mr, vr = [dev(p0) for _ in range(N)], [dev(m0) for _ in range(N)], [dev(v0) for _ in range(N)]
    gs = [torch.zeros(P, device="cuda") for _ in range(N)]
    cfg = dd.adam_cfg(step)
    keep = dd.ddppo_debug_peer_a8(ctx, mode, gd, pr, mr, vr, cfg, gs)
    torch.cuda.synchronize()
    ctx.check()
    del keep
    # fp32 rank-ordered sum, bit-exact
    ref = grads[0].clone()
    for x in grads[1:]:
        ref += x
    for r in range(N):
        lo, hi = (0, P) if mode == "allread" else _shard(P, N, r)
        assert torch.equal(gs[r][lo:hi].cpu(), ref[lo:hi]), (r, lo, hi)
    # parameters bit-identical on every rank
    p = [x.cpu() for x in pr]
    for r in range(1, N):
        assert torch.equal(p[r], p[0]), r
    # the oracle's clip 0.5 + Adam (fp64) on the mean of Eq. 3.  The mean is taken over the fp32 rank-ordered
    # sum checked bit-exactly above (the oracle's fp64 mean of fp32 inputs differs from it by fp32 rounding,
    # which the first Adam step amplifies without bound where |g| ~ eps)
    po, mo, vo, _ = optim.adam_step(p0.double().numpy(), ref.double().numpy() / N,
                                    m0.double().numpy(), v0.double().numpy(), step)
    d_gpu = p[0].double().numpy() - p0.double().numpy()
    d_ref = po - p0.double().numpy()
    err = np.abs(d_gpu - d_ref)
    assert np.all(err <= 1e-4 * np.abs(d_ref) + 1e-4 * np.abs(d_ref).max()), err.max()
    for r in range(N):
        lo, hi = (0, P) if mode == "allread" else _shard(P, N, r)
        for mine, oref in ((mr[r], mo), (vr[r], vo)):
            e = np.abs(mine[lo:hi].cpu().double().numpy() - oref[lo:hi])
            assert np.all(e <= 1e-4 * np.abs(oref[lo:hi]) + 1e-4 * np.abs(oref).max() + 1e-30), (r, e.max())


def test_peer_a8_modes_agree(ctx):
    """v1 and v2 differ only in the association order of the clip norm's fp64 partials."""
    N, P = 4, 200003
    g = torch.Generator().manual_seed(7)
    grads = [torch.randn(P, generator=g) for _ in range(N)]
    p0 = torch.randn(P, generator=g)
    out = {}
    for mode in ("allread", "sharded"):
        pr = [p0.clone().cuda() for _ in range(N)]
        z = [torch.zeros(P, device="cuda") for _ in range(3 * N)]
        dd.ddppo_debug_peer_a8(ctx, mode, [x.cuda() for x in grads], pr, z[:N], z[N:2 * N], dd.adam_cfg(1), z[2 * N:])
        torch.cuda.synchronize()
        out[mode] = pr[0].cpu()
    d = (out["allread"] - out["sharded"]).abs().max().item()
    assert d <= 1e-6 * 2.5e-4 * 10, d


@pytest.mark.parametrize("N", [2, 4, 8])
def test_peer_counts_emulated(ctx, N):
    rng = np.random.default_rng(N)
    vals = rng.integers(-(1 << 40), 1 << 40, size=(N, 7), dtype=np.int64)
    out = dd.ddppo_debug_peer_counts(ctx, vals)
    ctx.check()
    assert np.array_equal(out, np.broadcast_to(vals.sum(0), vals.shape))
    out2 = dd.ddppo_debug_peer_counts(ctx, vals[:, :1] * 3)  # a second epoch over fresh areas
    assert np.array_equal(out2[:, 0], np.full(N, 3 * vals[:, 0].sum()))
