"""Debug aid: per-face adaptive spectra, GPU (VB_ADAPTIVE_DUMP) vs oracle, on config 4 variants."""
import os
import sys

import numpy as np

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))


def main(n=16):
    dump = "gpurun_out/adaptive_dump_%d.txt" % n
    if os.path.exists(dump):
        os.remove(dump)
    os.environ["VB_ADAPTIVE_DUMP"] = dump
    import paper_2304_09770_b200 as vb
    from synthetic import make_problem
    from oracle.assemble import GlobalSystem
    from oracle.bddc import BDDC
    prob = make_problem("c4", n=n)
    ctx = vb.context_for(prob)
    ctx.factor()
    gs = GlobalSystem(prob)
    bd = BDDC(gs)
    gpu = {}
    for line in open(dump):
        v = line.split()
        gpu[int(v[0])] = np.sort(np.array([float(x) for x in v[2:]]))
    worst = []
    for e, lam in bd.adaptive_spectra.items():
        g = gpu.get(e)
        if g is None:
            print("face", e, "missing on GPU")
            continue
        lo = np.sort(lam)
        d = np.abs(g - lo).max() if g.size == lo.size else np.inf
        ns_o, ns_g = int((lo < 0.1).sum()), int((g < 0.1).sum())
        worst.append((d, e, ns_o, ns_g, lo[:3], g[:3], bd.ents[e].sharers))
    worst.sort(key=lambda t: -t[0])
    for w in worst[:15]:
        print("face %d maxdiff %.3e sel oracle %d gpu %d  oracle %s gpu %s sharers %s" % (w[1], w[0], w[2], w[3], w[4], w[5], w[6]))
    print("faces", len(worst), "total sel oracle", sum(w[2] for w in worst), "gpu", sum(w[3] for w in worst))


if __name__ == "__main__":
    main(int(sys.argv[1]) if len(sys.argv) > 1 else 16)
