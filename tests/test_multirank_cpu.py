"""Multi-rank bookkeeping on the CPU (no GPU): world-size 2 and 4 process groups over gloo.

Each process plays one rank of the weak-scaling box layouts of SURVEY §8(e) and asks the library's
host planner (vb_plan_exchange, the same counting that every multi-rank context checks its NCCL
transfers against) what it would send to and receive from every other rank.  The ranks exchange
those plans over gloo and check that they agree pairwise (what r sends p is what p expects from
r) for the three exchange modes, and that the owned free DOFs partition the global free vector."""
import os
import socket

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    port = s.getsockname()[1]
    s.close()
    return port


def _layout(vb, prob, rank_grid):
    """Subdomain -> rank: a box layout (tuple), a checkerboard over 2 ranks, or 3 ranks of which
    rank 2 owns no subdomain."""
    if isinstance(rank_grid, tuple):
        return vb.box_ranks(prob.sub_grid, rank_grid)
    sub = np.arange(int(np.prod(prob.sub_grid)))
    gx, gy, _ = prob.sub_grid
    i, j, k = sub % gx, (sub // gx) % gy, sub // (gx * gy)
    if rank_grid == "checker":
        return ((i + j + k) % 2).astype(np.int32)
    return (sub % 2).astype(np.int32)


def _world(rank_grid):
    return int(np.prod(rank_grid)) if isinstance(rank_grid, tuple) else {"checker": 2, "idle3": 3}[rank_grid]


def test_rank_without_subdomains_is_rejected():
    """Every rank must own at least one subdomain (include/vbddc.h, vb_setup): VB_EINVAL, named."""
    import paper_2304_09770_b200 as vb
    from synthetic import make_problem
    prob = make_problem("c1", n=8)
    srank = _layout(vb, prob, "idle3")
    snd, rcv, own = vb.plan_exchange(prob.mesh, prob.k, prob.cell_subdomain, srank, 0, 3, 0)
    assert own > 0
    with pytest.raises(vb.VBError) as e:
        vb.plan_exchange(prob.mesh, prob.k, prob.cell_subdomain, srank, 2, 3, 0)
    assert e.value.status == vb.VB_EINVAL and "owns no subdomain" in str(e.value)


def _worker(rank, world, port, name, kw, rank_grid, q):
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        import paper_2304_09770_b200 as vb
        from synthetic import make_problem
        prob = make_problem(name, **kw)
        srank = _layout(vb, prob, rank_grid)
        ok = True
        owned = None
        for mode in (0, 1, 2):
            snd, rcv, own = vb.plan_exchange(prob.mesh, prob.k, prob.cell_subdomain, srank, rank, world, mode)
            owned = own
            S = [torch.zeros(world, dtype=torch.int64) for _ in range(world)]
            Rv = [torch.zeros(world, dtype=torch.int64) for _ in range(world)]
            dist.all_gather(S, torch.tensor(snd))
            dist.all_gather(Rv, torch.tensor(rcv))
            S = torch.stack(S).numpy(); Rv = torch.stack(Rv).numpy()
            ok &= bool(np.array_equal(S, Rv.T))                      # send[r][p] == recv[p][r]
            ok &= bool(np.all(np.diag(S) == 0) and S.sum() > 0)
        O = [torch.zeros(1, dtype=torch.int64) for _ in range(world)]
        dist.all_gather(O, torch.tensor([owned]))
        total = int(sum(int(o.item()) for o in O))
        if rank == 0:
            from oracle.assemble import GlobalDofs   # the free DOF count of the oracle's numbering
            d = GlobalDofs(prob.mesh, prob.k)
            nfree = d.n_free_vel + d.npres
            q.put((ok, total, nfree))
    finally:
        dist.destroy_process_group()


@pytest.mark.parametrize("name,kw,rank_grid", [("c1", dict(n=8), (1, 1, 2)), ("c1", dict(n=8), (2, 2, 1)),
                                              ("c3", dict(n=8), (1, 2, 1)), ("c1", dict(n=8), (2, 2, 2)),
                                              ("c1", dict(n=8), "checker")])
def test_exchange_plans_agree_across_ranks(name, kw, rank_grid):
    world = _world(rank_grid)
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, world, port, name, kw, rank_grid, q)) for r in range(world)]
    for p in procs:
        p.start()
    for p in procs:
        p.join(300)
    assert all(p.exitcode == 0 for p in procs), [p.exitcode for p in procs]
    ok, total, nfree = q.get(timeout=10)
    assert ok
    assert total == nfree



def _cd_worker(rank, world, port, name, kw, rank_grid, q):
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        import paper_2304_09770_b200 as vb
        from synthetic import make_problem
        prob = make_problem(name, **kw)
        srank = _layout(vb, prob, rank_grid)
        p = vb.plan_coarse_dissection(prob.mesh, prob.k, prob.cell_subdomain, srank, rank, world)
        v = torch.tensor([p["n_interior"], p["n_S"], p["n_sep"], p["n_root"], p["n_primal"],
                          int(np.sum(srank == rank))])
        V = [torch.zeros(6, dtype=torch.int64) for _ in range(world)]
        dist.all_gather(V, v)
        if rank == 0:
            q.put((torch.stack(V).numpy(), int(np.prod(prob.sub_grid))))
    finally:
        dist.destroy_process_group()


@pytest.mark.parametrize("name,kw,rank_grid", [("c5", dict(dims=(32, 32, 64)), (1, 1, 2)),
                                              ("c1", dict(n=8), (2, 2, 1)),
                                              ("c1", dict(n=8), "checker")])
def test_coarse_dissection_plans_agree_across_ranks(name, kw, rank_grid):
    """SURVEY f1 host plan over gloo: every rank derives the same separator and root (the root is
    replicated), the interior sets and the separator partition the primal DOFs, the root is the
    separator plus one p_0 per subdomain, and each rank's root list holds its own p_0's.  c5 at its
    2-GPU size (1,024 subdomains): one cut plane of 8 x 8 subdomain faces."""
    world = _world(rank_grid)
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_cd_worker, args=(r, world, port, name, kw, rank_grid, q)) for r in range(world)]
    for p in procs:
        p.start()
    for p in procs:
        p.join(300)
    assert all(p.exitcode == 0 for p in procs), [p.exitcode for p in procs]
    V, nsub = q.get(timeout=10)
    nI, nS, nsep, nroot, npi, nown = V.T
    assert len(set(nsep)) == 1 and len(set(nroot)) == 1 and len(set(npi)) == 1
    assert nI.sum() + nsep[0] == npi[0]
    assert nroot[0] == nsep[0] + nsub
    assert np.all(nS >= nown) and np.all(nS - nown <= nsep[0])
    if rank_grid == "checker":
        assert np.all(nI == 0)             # every entity crosses ranks
    if name == "c5":
        # one cut plane z = 8 of the 8 x 8 x 16 subdomain grid: 64 faces, 2 * 8 * 7 edges, 7 * 7
        # vertices, 3 primal DOFs each; every other primal DOF is interior to one rank
        assert nsep[0] == 3 * (64 + 112 + 49)
        assert np.array_equal(nS, nsep + 512)


def test_coarse_dissection_plan_at_eight_gpus():
    """The 8-GPU sizes DESIGN.md §9 quotes, from the host planner on rank 0 of c5 at 64^3 cells
    (4,096 subdomains, 2x2x2 rank boxes): separator 3 (768 + 1,392 + 631) = 8,373 DOFs (three cut
    planes, inclusion-exclusion on their lines and centre point), root 8,373 + 4,096 = 12,469,
    8,589 interior DOFs per rank (= N_Pi of one 8^3-subdomain box)."""
    import paper_2304_09770_b200 as vb
    from synthetic import make_problem
    from synthetic.configs import C5_DIMS
    prob = make_problem("c5", dims=C5_DIMS[8])
    srank = vb.box_ranks(prob.sub_grid, (2, 2, 2))
    p = vb.plan_coarse_dissection(prob.mesh, prob.k, prob.cell_subdomain, srank, 0, 8)
    assert p["n_primal"] + 4096 == 81181          # N_c at 8 GPUs
    assert p["n_sep"] == 8373 and p["n_root"] == 12469
    assert p["n_interior"] == 8589
    assert p["n_S"] == 2675 and p["n_local"] == 8608 + 2675   # 2,163 touched separator DOFs + 512 p_0
    print("8-GPU plan rank 0:", p)
