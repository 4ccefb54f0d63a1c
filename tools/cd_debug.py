"""Debug of the coarse dissection (f1): dumps (VB_CD_DUMP) of the dense coarse matrix of a 1-rank run
and the local/root matrices of an R-rank loopback run, compared in numpy."""
import os
import sys
import concurrent.futures as cf
import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2304_09770_b200 as vb  # noqa: E402
from synthetic import make_problem  # noqa: E402

D = os.environ.setdefault("VB_CD_DUMP", "gpurun_out/cd")
os.makedirs(D, exist_ok=True)


def load(name, r=0):
    a = np.fromfile(os.path.join(D, "%s_r%d.bin" % (name, r)), dtype=np.int64, count=2)
    rows, cols = int(a[0]), int(a[1])
    if name in ("Iglob", "Sglob", "root"):
        return np.fromfile(os.path.join(D, "%s_r%d.bin" % (name, r)), dtype=np.int64)[2:]
    return np.fromfile(os.path.join(D, "%s_r%d.bin" % (name, r)), dtype=np.float64)[2:].reshape(cols, rows).T


prob = make_problem("c1", n=8)
grid = (1, 2, 2)
R = 4
srank = vb.box_ranks(prob.sub_grid, grid)


def run(opt):
    world = vb.LoopbackWorld(R)
    streams = [torch.cuda.Stream() for _ in range(R)]

    def main(r):
        c = vb.context_for(prob, stream=streams[r], rank=r, nranks=R, subdomain_rank=srank, world=world)
        c.set_option("coarse_dissection", opt)
        try:
            c.factor()
            return "ok"
        except Exception as e:
            return str(e)
        finally:
            c.close()

    with cf.ThreadPoolExecutor(R) as ex:
        print(list(ex.map(main, range(R))))
    world.close()


run(0)   # dense coarse on 4 ranks: kc in the 4-rank numbering
Kc = load("kc")
run(1)
Nc = Kc.shape[0]
print("Nc", Nc, "sym", np.abs(Kc - Kc.T).max())
root = load("root")
print("root", root.size)
Kr = load("kroot")
# expected root: Schur complement of Kc onto root
mask = np.zeros(Nc, bool)
mask[root] = True
I = np.where(~mask)[0]
A = Kc[np.ix_(I, I)]
print("interior count", I.size, "min eig interior", np.linalg.eigvalsh(A).min())
S = Kc[np.ix_(root, root)] - Kc[np.ix_(root, I)] @ np.linalg.solve(A, Kc[np.ix_(I, root)])
Krs = np.tril(Kr) + np.tril(Kr, -1).T
print("root vs Schur: max diff %.3e (max %.3e)" % (np.abs(Krs - S).max(), np.abs(S).max()))
nsep = root.size - int(np.prod(prob.sub_grid))
print("nsep", nsep, "min eig root vel", np.linalg.eigvalsh(Krs[:nsep, :nsep]).min(), "expected", np.linalg.eigvalsh(S[:nsep, :nsep]).min())
for r in range(R):
    Ig, Sg = load("Iglob", r), load("Sglob", r)
    K = load("kloc", r)
    nI = Ig.size
    nIp = (nI + 31) // 32 * 32
    loc = np.concatenate([Ig, Sg])
    pos = np.concatenate([np.arange(nI), nIp + np.arange(Sg.size)])
    Kl = K[np.ix_(pos, pos)]
    Ke = Kc[np.ix_(loc, loc)]
    dII = np.abs(Kl[:nI, :nI] - Ke[:nI, :nI]).max()
    dIS = np.abs(Kl[nI:, :nI] - Ke[nI:, :nI]).max()
    print("rank %d nI %d nS %d: II diff %.3e IS diff %.3e (scale %.3e)" % (r, nI, Sg.size, dII, dIS, np.abs(Ke).max()))
    Dm = np.abs(Kl[nI:, :nI] - Ke[nI:, :nI])
    bad = np.argwhere(Dm > 1e-12)
    print("   bad IS entries", bad.shape[0], "of", Dm.size, "; rows (S index):", np.unique(bad[:, 0])[:20], "glob", Sg[np.unique(bad[:, 0])[:10]])
    print("   cols (I index):", np.unique(bad[:, 1])[:20], "glob", Ig[np.unique(bad[:, 1])[:10]])
    print("   sample local vs dense:", [(Kl[nI + a, b], Ke[nI + a, b]) for a, b in bad[:3]])
    NPi = Nc - int(np.prod(prob.sub_grid))
    print("   NPi", NPi, "S p0 count", int((Sg >= NPi).sum()))
    P = load("piece", r)[:Sg.size, :Sg.size]
    Kd = Kl[:nI, :nI]
    Sexp = Kl[nI:, nI:] - Kl[nI:, :nI] @ np.linalg.solve(Kd, Kl[:nI, nI:])
    print("   piece vs local Schur %.3e" % np.abs(P - Sexp).max())
