"""Stress the triangular-K-skip GEMM path (vb_debug_gemm kz) against torch, repeated, including the
distributed coarse row-block shape (A = W[lo:, lo:]^T, B = W[lo:, :hi], kzB = -lo)."""
import os
import sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))


def colmajor(X):
    return X.transpose(-1, -2).contiguous()


def main():
    import torch
    import paper_2304_09770_b200 as vb
    bad = 0
    for rep in range(40):
        n = [300, 517, 1100][rep % 3]
        g = torch.Generator(device="cuda").manual_seed(rep)
        W = torch.tril(torch.randn(n, n, dtype=torch.float64, device="cuda", generator=g))
        d = torch.rand(n, dtype=torch.float64, device="cuda", generator=g) + 0.5
        R = [2, 3, 8][rep % 3]
        rows = (n + R - 1) // R
        for r in range(R):
            lo, hi = r * rows, min(n, (r + 1) * rows)
            if lo >= hi:
                continue
            ref = (W[lo:, lo:hi].T * d[lo:]) @ W[lo:, :hi]            # mine x hi
            A = colmajor(W[lo:, lo:hi]).reshape(1, hi - lo, n - lo)   # stored A = W[lo:, lo:hi] (K x mine)
            B = colmajor(W[lo:, :hi]).reshape(1, hi, n - lo)          # stored B = W[lo:, :hi] (K x hi)
            C = torch.zeros(1, hi, hi - lo, dtype=torch.float64, device="cuda")
            vb.debug_gemm(A, B, C, d=d[lo:].contiguous(), transA=True, kz=(0, -lo))
            err = (C[0].T - ref).abs().max().item()
            if err > 1e-11 * ref.abs().max().item():
                bad += 1
                print("mismatch rep", rep, "n", n, "R", R, "r", r, "err", err, flush=True)
    print("bad", bad)


if __name__ == "__main__":
    main()
