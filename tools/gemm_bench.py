"""DMMA GEMM of the factorisation (vb_debug_gemm) vs torch float64 matmul (cuBLAS DGEMM) on the
shapes the factor runs: one large square problem (dense 2-D grid path) and batched per-subdomain
trailing updates / products (tile-list path).  TFLOP/s against the measured DMMA peak 37.2."""
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))


def bench(fn, reps=3):
    import torch
    fn()
    torch.cuda.synchronize()
    best = 1e30
    for _ in range(reps):
        t = time.perf_counter()
        fn()
        torch.cuda.synchronize()
        best = min(best, time.perf_counter() - t)
    return best


def main():
    import torch
    import paper_2304_09770_b200 as vb
    cases = [(8192, 8192, 8192, 1), (1285, 1285, 128, 512), (1158, 1158, 1285, 64), (1080, 1080, 1080, 128),
             (1285, 128, 128, 512)]
    for M, N, K, b in cases:
        A = torch.randn(b, K, M, dtype=torch.float64, device="cuda")   # column-major M x K
        B = torch.randn(b, N, K, dtype=torch.float64, device="cuda")   # column-major K x N
        C = torch.zeros(b, N, M, dtype=torch.float64, device="cuda")
        f = 2.0 * M * N * K * b
        t1 = bench(lambda: vb.debug_gemm(A, B, C))
        At, Bt = A.transpose(1, 2), B.transpose(1, 2)
        t2 = bench(lambda: torch.bmm(At, Bt))
        print("M=%5d N=%5d K=%5d batch=%4d   vb DMMA %6.2f TF/s (%.0f%% of 37.2)   cuBLAS %6.2f TF/s" %
              (M, N, K, b, f / t1 / 1e12, 100 * f / t1 / 1e12 / 37.2, f / t2 / 1e12), flush=True)


if __name__ == "__main__":
    main()
