"""One shape of the factorisation's DMMA GEMM (vb_debug_gemm), for ncu captures and A/B timing:
  python tools/gemm_one.py M N K batch [transA transB lower_scaled]"""
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))


def main():
    import torch
    import paper_2304_09770_b200 as vb
    M, N, K, b = [int(x) for x in sys.argv[1:5]]
    tA, tB = (int(sys.argv[5]), int(sys.argv[6])) if len(sys.argv) > 6 else (0, 0)
    scaled = len(sys.argv) > 7 and int(sys.argv[7])
    A = torch.randn(b, M if tA else K, K if tA else M, dtype=torch.float64, device="cuda")
    B = torch.randn(b, K if tB else N, N if tB else K, dtype=torch.float64, device="cuda")
    C = torch.zeros(b, N, M, dtype=torch.float64, device="cuda")
    d = torch.rand(K, dtype=torch.float64, device="cuda") if scaled else None
    f = 2.0 * M * N * K * b
    vb.debug_gemm(A, B, C, d=d, transA=bool(tA), transB=bool(tB))
    torch.cuda.synchronize()
    best = 1e30
    for _ in range(int(os.environ.get("REPS", "5"))):
        t = time.perf_counter()
        vb.debug_gemm(A, B, C, d=d, transA=bool(tA), transB=bool(tB))
        torch.cuda.synchronize()
        best = min(best, time.perf_counter() - t)
    print("M=%d N=%d K=%d batch=%d tA=%d tB=%d scaled=%d: %.2f TF/s (%.0f%% of 37.2)" %
          (M, N, K, b, tA, tB, int(bool(scaled)), f / best / 1e12, 100 * f / best / 1e12 / 37.2), flush=True)


if __name__ == "__main__":
    main()
