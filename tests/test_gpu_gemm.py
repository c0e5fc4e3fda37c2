"""The tcgen05 GEMM used by the backward (weight/input gradients), through its diagnostic C entry.

Reference: the plain definition C = A B^T on the bf16-rounded operands, accumulated in fp64
(torch CPU rounding to bf16 = round-to-nearest-even, the same rounding the kernel's staging
uses); tolerance covers fp32 accumulation only."""
import numpy as np
import pytest
import torch

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


def _bf(x):
    return torch.from_numpy(x).to(torch.bfloat16).double().numpy()


@pytest.mark.parametrize("M,N,K,a_kmajor,b_kmajor,splits", [
    (128, 128, 64, True, True, 1), (128, 32, 16, True, True, 1), (100, 37, 70, True, False, 1),
    (1536, 512, 256, False, False, 1),   # dW_hh = dG_h^T H_in  (both operands sample-major in HBM)
    (1536, 64, 256, False, False, 1),    # dW_ih = dG_x^T X
    (256, 64, 1536, True, False, 1),     # dX = dG_x W_ih
    (300, 200, 130, False, True, 1),
    (32, 288, 16384, False, False, 16),  # conv wgrad: K = output pixels, split-K
    (64, 576, 5000, False, True, 7)])
def test_gemm_tc(dd, ctx, M, N, K, a_kmajor, b_kmajor, splits):
    rng = np.random.default_rng(M * 7 + N * 3 + K)
    A = rng.normal(size=(M, K)).astype(np.float32)
    B = rng.normal(size=(N, K)).astype(np.float32)
    # store A either [M][K] (k contiguous) or [K][M] (m contiguous); same for B
    Ast = A if a_kmajor else np.ascontiguousarray(A.T)
    Bst = B if b_kmajor else np.ascontiguousarray(B.T)
    sam, sak = (K, 1) if a_kmajor else (1, M)
    sbn, sbk = (K, 1) if b_kmajor else (1, N)
    C = torch.full((M, N), 123.0, device="cuda")
    part = torch.zeros(splits * M * N, device="cuda") if splits > 1 else None
    dd.ddppo_debug_gemm_bf16(ctx, torch.from_numpy(Ast).cuda(), sam, sak, torch.from_numpy(Bst).cuda(), sbn, sbk, C,
                             N, M, N, K, splits, part)
    torch.cuda.synchronize()
    ref = _bf(A) @ _bf(B).T
    got = C.cpu().numpy()
    err = np.abs(got - ref).max()
    scale = np.abs(_bf(A)) @ np.abs(_bf(B)).T
    assert err <= 1e-5 * scale.max() + 1e-6, (err, scale.max())


@pytest.mark.parametrize("M,N,K,a_kmajor,b_kmajor,splits", [
    (128, 64, 64, True, True, 1), (300, 200, 130, False, True, 1), (4096, 32, 49, True, True, 1),
    (64, 576, 5000, False, True, 7)])
def test_gemm_tc_split_precision(dd, ctx, M, N, K, a_kmajor, b_kmajor, splits):
    """prec = 3 (bf16x3): against the fp64 product of the UNROUNDED fp32 operands; the error bound
    is that of fp32-level operands (2^-16 relative per term) plus fp32 accumulation."""
    rng = np.random.default_rng(M + N + K)
    A = rng.normal(size=(M, K)).astype(np.float32)
    B = rng.normal(size=(N, K)).astype(np.float32)
    Ast = A if a_kmajor else np.ascontiguousarray(A.T)
    Bst = B if b_kmajor else np.ascontiguousarray(B.T)
    sam, sak = (K, 1) if a_kmajor else (1, M)
    sbn, sbk = (K, 1) if b_kmajor else (1, N)
    C = torch.full((M, N), 123.0, device="cuda")
    part = torch.zeros(splits * M * N, device="cuda") if splits > 1 else None
    dd.ddppo_debug_gemm_bf16(ctx, torch.from_numpy(Ast).cuda(), sam, sak, torch.from_numpy(Bst).cuda(), sbn, sbk, C,
                             N, M, N, K, splits, part, prec=3)
    torch.cuda.synchronize()
    ref = A.astype(np.float64) @ B.astype(np.float64).T
    err = np.abs(C.cpu().numpy() - ref).max()
    scale = np.abs(A.astype(np.float64)) @ np.abs(B.astype(np.float64)).T
    assert err <= 3e-5 * scale.max(), (err, scale.max())
    # and it is really more accurate than plain bf16 operands
    C1 = torch.zeros((M, N), device="cuda")
    dd.ddppo_debug_gemm_bf16(ctx, torch.from_numpy(Ast).cuda(), sam, sak, torch.from_numpy(Bst).cuda(), sbn, sbk, C1,
                             N, M, N, K, splits, part, prec=1)
    torch.cuda.synchronize()
    assert err * 20 < np.abs(C1.cpu().numpy() - ref).max()
