"""The factorisation's grouped DMMA GEMM (dense.cu, used by A1-A5) against torch float64 matmul:
all transpose cases, diagonal scaling, beta accumulation, ragged sizes that span several
64 x 64 x 16 tiles with partial edge tiles (odd leading dimensions: 8-byte copy path; even: 16-byte), batched problems and the large-problem 2-D grid path."""
import pytest

pytestmark = pytest.mark.gpu


def _colmajor(X):
    return X.transpose(-1, -2).contiguous()


@pytest.mark.parametrize("M,N,K,batch", [(1, 1, 1, 1), (37, 5, 3, 2), (130, 70, 33, 3), (257, 129, 200, 4),
                                         (1285, 1158, 129, 2), (9001, 4097, 70, 1)])
@pytest.mark.parametrize("tA,tB", [(False, False), (True, False), (False, True), (True, True)])
def test_gemm_vs_torch(M, N, K, batch, tA, tB):
    import torch
    import paper_2304_09770_b200 as vb
    if M * N > 4e6 and (tA or tB):
        pytest.skip("large case: one transpose combination is enough")
    g = torch.Generator(device="cuda").manual_seed(M * 7 + N * 3 + K)
    A = torch.randn(batch, K if tA else M, M if tA else K, dtype=torch.float64, device="cuda", generator=g)
    B = torch.randn(batch, N if tB else K, K if tB else N, dtype=torch.float64, device="cuda", generator=g)
    C0 = torch.randn(batch, M, N, dtype=torch.float64, device="cuda", generator=g)
    d = torch.rand(K, dtype=torch.float64, device="cuda", generator=g) + 0.5
    opA = A.transpose(1, 2) if tA else A
    opB = B.transpose(1, 2) if tB else B
    ref = -0.5 * (opA * d) @ opB + 2.0 * C0
    C = _colmajor(C0)
    vb.debug_gemm(_colmajor(A), _colmajor(B), C, alpha=-0.5, beta=2.0, d=d, transA=tA, transB=tB)
    got = C.transpose(1, 2)
    err = (got - ref).abs().max().item()
    scale = ((opA.abs() * d) @ opB.abs()).max().item()
    assert err <= 1e-14 * K * scale + 1e-13, err


@pytest.mark.parametrize("n,batch", [(70, 3), (300, 2), (1300, 1)])
def test_gemm_triangular_skip(n, batch):
    """Triangular-operand K skipping (GemmProb.kz_on, used for W^T D W with W = L^-1 lower): the
    kernel starts each tile's K loop at its first non-zero slab; the result must equal the full
    product (the skipped slabs are exactly zero)."""
    import torch
    import paper_2304_09770_b200 as vb
    g = torch.Generator(device="cuda").manual_seed(n)
    W = torch.tril(torch.randn(batch, n, n, dtype=torch.float64, device="cuda", generator=g))
    d = torch.rand(n, dtype=torch.float64, device="cuda", generator=g) + 0.5
    ref = (W.transpose(1, 2) * d) @ W
    C = torch.zeros(batch, n, n, dtype=torch.float64, device="cuda")
    Wc = _colmajor(W)
    vb.debug_gemm(Wc, Wc, C, d=d, transA=True, kz=(0, 0))
    got = C.transpose(1, 2)
    assert (got - ref).abs().max().item() <= 1e-12 * ref.abs().max().item()
