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


@pytest.mark.parametrize("M,N,K,a_kmajor,b_kmajor", [
    (128, 128, 64, True, True), (128, 32, 16, True, True), (100, 37, 70, True, False),
    (1536, 512, 256, False, False),   # dW_hh = dG_h^T H_in  (both operands sample-major in HBM)
    (1536, 64, 256, False, False),    # dW_ih = dG_x^T X
    (256, 64, 1536, True, False),     # dX = dG_x W_ih
    (300, 200, 130, False, True)])
def test_gemm_tc(dd, ctx, M, N, K, a_kmajor, b_kmajor):
    rng = np.random.default_rng(M * 7 + N * 3 + K)
    A = rng.normal(size=(M, K)).astype(np.float32)
    B = rng.normal(size=(N, K)).astype(np.float32)
    # store A either [M][K] (k contiguous) or [K][M] (m contiguous); same for B
    Ast = A if a_kmajor else np.ascontiguousarray(A.T)
    Bst = B if b_kmajor else np.ascontiguousarray(B.T)
    sam, sak = (K, 1) if a_kmajor else (1, M)
    sbn, sbk = (K, 1) if b_kmajor else (1, N)
    C = torch.full((M, N), 123.0, device="cuda")
    dd.ddppo_debug_gemm_bf16(ctx, torch.from_numpy(Ast).cuda(), sam, sak, torch.from_numpy(Bst).cuda(), sbn, sbk, C,
                             N, M, N, K)
    torch.cuda.synchronize()
    ref = _bf(A) @ _bf(B).T
    got = C.cpu().numpy()
    err = np.abs(got - ref).max()
    scale = np.abs(_bf(A)) @ np.abs(_bf(B)).T
    assert err <= 1e-5 * scale.max() + 1e-6, (err, scale.max())
