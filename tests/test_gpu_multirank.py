"""Multi-rank data path on ONE GPU through the loopback transport: R library ranks
run as R threads of this process, each owning a box of subdomains, exchanging interface sums (C1),
coarse pieces (C2), dot partials (C3) and local coarse matrices (C4) by host-synchronised device
copies -- the same exchange plans the NCCL transport runs over NVLink.  Gates: the R-rank solve
equals the oracle (SURVEY §8(c) parity gates) and the 1-rank solve (decomposition invariance:
iterations equal, solution to 1e-12)."""
import concurrent.futures as cf

import numpy as np
import pytest

from synthetic import make_problem

pytestmark = pytest.mark.gpu


def _run_ranks(prob, rank_grid, rtol=1e-10, check_operator=True, srank=None, R=None, p2p=False, coarse=None,
               blocks=None):
    import torch
    import paper_2304_09770_b200 as vb
    if srank is None:
        R = int(np.prod(rank_grid))
        srank = vb.box_ranks(prob.sub_grid, rank_grid)
    world = vb.LoopbackWorld(R)
    streams = [torch.cuda.Stream() for _ in range(R)]

    def rank_main(r):
        ctx = vb.context_for(prob, stream=streams[r], rank=r, nranks=R, subdomain_rank=srank, world=world)
        if p2p:
            ctx.set_option("p2p", 1)
        if coarse is not None:
            ctx.set_option("coarse_dissection", coarse)
        if blocks is not None:
            ctx.set_option("coarse_blocks", blocks)
        ctx.factor()
        stats = ctx.stats()
        rhs = torch.zeros(ctx.n_free, dtype=torch.float64, device="cuda")
        x = torch.zeros_like(rhs)
        torch.cuda.synchronize()
        ctx.build_rhs(vb.problem_args(prob), rhs)
        rep = ctx.pcg_solve(rhs, x, rtol=rtol)
        res = None
        if check_operator:
            y = torch.zeros_like(rhs)
            ctx.apply_operator(x, y)
            res = (rhs - y).cpu().numpy()
        # the host-buffer entry point on the same rank-local layout (vb_pcg_solve_host: owned DOFs)
        rh = rhs.cpu().numpy()
        xh = np.zeros(ctx.n_free)
        ctx.pcg_solve_host(rh, xh, rtol=rtol)
        out = dict(rep=rep, ids=ctx.dof_layout(), x=x.cpu().numpy(), rhs=rh, res=res, x_host=xh, stats=stats)
        ctx.close()
        return out

    def guarded(r):
        try:
            return rank_main(r)
        except Exception as e:   # keep every rank's error: the first failure aborts the others
            return e

    with cf.ThreadPoolExecutor(R) as ex:
        outs = list(ex.map(guarded, range(R)))
    world.close()
    errs = [(r, o) for r, o in enumerate(outs) if isinstance(o, Exception)]
    assert not errs, "rank errors: " + "; ".join("rank %d: %s" % (r, e) for r, e in errs)
    return outs


def _assemble(outs, n_total):
    x = np.full(n_total, np.nan)
    b = np.full(n_total, np.nan)
    for o in outs:
        x[o["ids"]] = o["x"]
        b[o["ids"]] = o["rhs"]
    return x, b


def _global_free_ids(gs):
    return np.concatenate([gs.dofs.free_vel, gs.dofs.nvel + np.arange(gs.dofs.npres)])


@pytest.mark.parametrize("name,kw,rank_grid", [
    ("c1", {}, (1, 1, 2)),
    ("c1", {}, (2, 2, 2)),
    ("c1", dict(n=8), (1, 2, 2)),
    ("c1", dict(n=8), (2, 2, 2)),
    ("c4", dict(n=8, constraints=dict(adaptive_tau=0.0)), (2, 1, 1)),
    ("c3", dict(n=8), (2, 1, 1)),
])
def test_multirank_matches_oracle_and_single_rank(name, kw, rank_grid):
    import torch
    import paper_2304_09770_b200 as vb
    from oracle.assemble import GlobalSystem
    from oracle.bddc import BDDC
    prob = make_problem(name, **kw)
    gs = GlobalSystem(prob)
    u_o, p_o, rep_o = BDDC(gs).solve(rtol=1e-10)
    # single rank reference
    ctx = vb.context_for(prob)
    ctx.factor()
    rhs1 = torch.zeros(ctx.n_free, dtype=torch.float64, device="cuda")
    ctx.build_rhs(vb.problem_args(prob), rhs1)
    x1 = torch.zeros_like(rhs1)
    rep1 = ctx.pcg_solve(rhs1, x1, rtol=1e-10)
    ids1 = ctx.dof_layout()
    x1 = x1.cpu().numpy()
    outs = _run_ranks(prob, rank_grid)
    gid = _global_free_ids(gs)
    for o in outs:      # vb_pcg_solve_host == vb_pcg_solve on every rank (owned-DOF sizes)
        assert np.abs(o["x_host"] - o["x"]).max() <= 1e-14 * np.abs(o["x"]).max()
    assert np.array_equal(np.sort(np.concatenate([o["ids"] for o in outs])), np.sort(gid))   # a partition
    pos = {int(g): i for i, g in enumerate(gid)}
    n = gid.size
    xR, bR = _assemble([dict(o, ids=np.array([pos[int(g)] for g in o["ids"]])) for o in outs], n)
    assert np.array_equal(ids1, gid)
    # the distributed rhs assembly equals the single-rank one
    assert np.abs(bR - rhs1.cpu().numpy()).max() <= 1e-13 * np.abs(bR).max()
    for o in outs:
        # dot partials are summed per rank: counts within +-1, the non-enriched sinker
        # case (kappa ~ 270, ~86 iterations) included
        assert abs(o["rep"]["iterations"] - rep1["iterations"]) <= 1, (o["rep"]["iterations"], rep1["iterations"])
        # reductions run in a different order than on one rank: kappa to rounding of the Lanczos
        # coefficients (the sinker case without enrichment has kappa ~ 270)
        assert abs(o["rep"]["kappa"] - rep1["kappa"]) <= 1e-4 * rep1["kappa"]
        assert o["rep"]["n_primal"] == rep1["n_primal"]
    # not bitwise (dot partials are summed per rank): both are rtol-1e-10 solutions
    assert np.linalg.norm(xR - x1) <= 1e-10 * np.linalg.norm(x1)
    nv = gs.dofs.n_free_vel
    assert np.linalg.norm(xR[:nv] - u_o) <= 1e-8 * np.linalg.norm(u_o)
    assert np.linalg.norm(xR[nv:] - p_o) <= 1e-8 * np.linalg.norm(p_o)
    assert abs(outs[0]["rep"]["iterations"] - rep_o["iterations"]) <= 1, (outs[0]["rep"]["iterations"], rep_o["iterations"])
    # true residual of the distributed element-by-element operator
    rR = np.concatenate([o["res"] for o in outs])
    assert np.linalg.norm(rR) <= 1e-8 * np.linalg.norm(bR)


@pytest.mark.parametrize("n,rank_grid", [(8, (2, 1, 1)), (16, (2, 2, 1))])
def test_multirank_adaptive(n, rank_grid):
    """Adaptive enrichment across rank boundaries: faces shared by two ranks are solved redundantly
    (bitwise-identical inputs), so the primal space and the iterates match the single-rank run;
    n = 16 has floating subdomains (singular face Schur complements, DESIGN A28) on the cut."""
    import torch
    import paper_2304_09770_b200 as vb
    prob = make_problem("c4", n=n)
    ctx = vb.context_for(prob)
    ctx.factor()
    rhs1 = torch.zeros(ctx.n_free, dtype=torch.float64, device="cuda")
    ctx.build_rhs(vb.problem_args(prob), rhs1)
    x1 = torch.zeros_like(rhs1)
    rep1 = ctx.pcg_solve(rhs1, x1, rtol=1e-10)
    outs = _run_ranks(prob, rank_grid, check_operator=False)
    for o in outs:
        assert o["rep"]["n_adaptive"] == rep1["n_adaptive"]
        assert o["rep"]["n_primal"] == rep1["n_primal"]
        assert o["rep"]["iterations"] == rep1["iterations"]


@pytest.mark.parametrize("assign", ["checkerboard", "stripes3"])
def test_multirank_irregular_assignment(assign):
    """Non-box subdomain-to-rank maps: a checkerboard (every interface entity crosses ranks; vertices
    shared by 8 subdomains on 2 ranks) and 3 ranks owning interleaved x-stripes (ragged rank sizes,
    every rank pair adjacent).  Same gates as above against the 1-rank solve."""
    import torch
    import paper_2304_09770_b200 as vb
    prob = make_problem("c1", n=8)
    sub = np.arange(int(np.prod(prob.sub_grid)))
    gx, gy, gz = prob.sub_grid
    i, j, k = sub % gx, (sub // gx) % gy, sub // (gx * gy)
    if assign == "checkerboard":
        srank, R = ((i + j + k) % 2).astype(np.int32), 2
    else:
        srank, R = (i % 3).astype(np.int32), 3
    ctx = vb.context_for(prob)
    ctx.factor()
    rhs1 = torch.zeros(ctx.n_free, dtype=torch.float64, device="cuda")
    ctx.build_rhs(vb.problem_args(prob), rhs1)
    x1 = torch.zeros_like(rhs1)
    rep1 = ctx.pcg_solve(rhs1, x1, rtol=1e-10)
    ids1 = ctx.dof_layout()
    x1 = x1.cpu().numpy()
    outs = _run_ranks(prob, None, srank=srank, R=R)
    ids = np.concatenate([o["ids"] for o in outs])
    assert np.array_equal(np.sort(ids), np.sort(ids1))
    pos = {int(g): q for q, g in enumerate(ids1)}
    xR = np.full(ids1.size, np.nan)
    for o in outs:
        xR[[pos[int(g)] for g in o["ids"]]] = o["x"]
    for o in outs:
        assert abs(o["rep"]["iterations"] - rep1["iterations"]) <= 1
        assert abs(o["rep"]["kappa"] - rep1["kappa"]) <= 1e-4 * rep1["kappa"]
    assert np.linalg.norm(xR - x1) <= 1e-10 * np.linalg.norm(x1)
    rR = np.concatenate([o["res"] for o in outs])
    assert np.linalg.norm(rR) <= 1e-8 * np.linalg.norm(rhs1.cpu().numpy())


def _srank(prob, assign):
    sub = np.arange(int(np.prod(prob.sub_grid)))
    gx, gy, _ = prob.sub_grid
    i, j, k = sub % gx, (sub // gx) % gy, sub // (gx * gy)
    if assign == "checkerboard":
        return ((i + j + k) % 2).astype(np.int32), 2
    return (i % 3).astype(np.int32), 3


@pytest.mark.parametrize("name,kw,assign", [
    ("c1", {}, (2, 2, 2)),
    ("c1", dict(n=8), "checkerboard"),
    ("c1", dict(n=8), "stripes3"),
    ("c3", dict(n=8), (2, 1, 1)),
])
def test_multirank_peer_stores_bitwise(name, kw, assign):
    """Option "p2p": the two per-step interface exchanges (S^ p copies, extension products) are
    stores from the producing kernels straight into the peers' receive areas plus a barrier.  The
    receive areas get the same values at the same positions as through pack + send/recv, so the
    solve is bitwise identical to the default path (entities shared by up to 8 subdomains on 2
    ranks, and 3 ranks that all neighbour each other, included)."""
    import paper_2304_09770_b200 as vb
    prob = make_problem(name, **kw)
    if isinstance(assign, tuple):
        srank, R = None, None
        grid = assign
    else:
        (srank, R), grid = _srank(prob, assign), None
    base = _run_ranks(prob, grid, srank=srank, R=R, check_operator=False)
    peer = _run_ranks(prob, grid, srank=srank, R=R, check_operator=False, p2p=True)
    for a, b in zip(base, peer):
        assert a["rep"]["iterations"] == b["rep"]["iterations"]
        assert np.array_equal(a["ids"], b["ids"])
        assert np.array_equal(a["x"], b["x"])
        assert np.array_equal(a["x_host"], b["x_host"])
        assert a["rep"]["rel_residual"] == b["rep"]["rel_residual"]


@pytest.mark.parametrize("name,kw,grid", [
    ("c1", dict(n=8), 1),                 # one rank, one part: root = the p_0's only
    ("c1", dict(n=8), "blocks8"),         # one rank, 8 blocks of 2^3 subdomains (RCB)
    ("c2", {}, "blocks8"),                # 64 subdomains in 8 blocks
    ("c4", dict(n=16, constraints=dict(adaptive_tau=2.0)), "blocks4"),   # adaptive rows, 4 blocks
    ("c3", dict(n=8), "blocks2"),         # k = 3, 2 blocks
    ("c1", dict(n=8), (2, 2, 2)),         # 8 rank boxes of 2^3 subdomains (interior entities on every rank)
    ("c1", dict(n=8), "checkerboard"),    # every entity crosses ranks: no interior DOFs anywhere
    ("c1", dict(n=8), "stripes3"),        # ragged rank sizes
    ("c3", dict(n=8), (2, 1, 1)),         # k = 3, jittered triangulated cells
    ("c1", dict(n=8), ((1, 1, 2), 2)),    # two levels: 2 ranks x 2 blocks of 16 subdomains
    ("c2", {}, ((2, 2, 2), 2)),           # 8 ranks x 2 blocks
    ("c4", dict(n=16, constraints=dict(adaptive_tau=2.0)), ((2, 1, 1), 4)),   # adaptive, 4 blocks per rank
    ("c4", dict(n=16, constraints=dict(adaptive_tau=2.0)), (2, 2, 1)),   # adaptive rows on the separator
])
def test_coarse_dissection_matches_dense_coarse(name, kw, grid):
    """the rank-level dissection of the coarse saddle problem (block elimination of every
    rank's interior primal DOFs, root = separator + p_0) gives the solve of the
    replicated dense coarse inverse up to rounding: iterations within 1, kappa to 1e-4, solutions to 1e-10;
    its root is smaller than N_c whenever a rank owns interior entities."""
    import torch
    import paper_2304_09770_b200 as vb
    prob = make_problem(name, **kw)
    if grid == 1 or str(grid).startswith("blocks"):
        blocks = 1 if grid == 1 else int(grid[6:])
        runs = []
        for opt in (0, 1):
            ctx = vb.context_for(prob)
            ctx.set_option("coarse_dissection", opt)
            ctx.set_option("coarse_blocks", blocks)
            ctx.factor()
            st = ctx.stats()
            rhs = torch.zeros(ctx.n_free, dtype=torch.float64, device="cuda")
            ctx.build_rhs(vb.problem_args(prob), rhs)
            x = torch.zeros_like(rhs)
            rep = ctx.pcg_solve(rhs, x, rtol=1e-10)
            runs.append([dict(rep=rep, x=x.cpu().numpy(), ids=ctx.dof_layout(), stats=st)])
            ctx.close()
        n_sub = int(np.prod(prob.sub_grid))
        if blocks == 1:
            assert runs[1][0]["stats"]["n_coarse_root"] == n_sub      # only the p_0's
        else:
            assert n_sub < runs[1][0]["stats"]["n_coarse_root"] < runs[1][0]["stats"]["n_coarse"]
        assert runs[0][0]["stats"]["n_coarse_root"] == 0
    else:
        if isinstance(grid, str):
            srank, R = _srank(prob, grid)
            runs = [_run_ranks(prob, None, srank=srank, R=R, coarse=opt, check_operator=False) for opt in (0, 1)]
        elif isinstance(grid[0], tuple):   # two levels: (rank grid, blocks per rank)
            runs = [_run_ranks(prob, grid[0], coarse=opt, blocks=grid[1] if opt else None, check_operator=False)
                    for opt in (0, 1)]
        else:
            runs = [_run_ranks(prob, grid, coarse=opt, check_operator=False) for opt in (0, 1)]
    dense, dis = runs
    for a, b in zip(dense, dis):
        assert np.array_equal(a["ids"], b["ids"])
        assert abs(a["rep"]["iterations"] - b["rep"]["iterations"]) <= 1
        assert abs(a["rep"]["kappa"] - b["rep"]["kappa"]) <= 1e-4 * a["rep"]["kappa"]
        assert a["rep"]["n_coarse"] == b["rep"]["n_coarse"]
        st = b["stats"]
        assert 0 < st["n_coarse_root"] <= st["n_coarse"]
        if grid == (2, 2, 2):
            assert st["n_coarse_root"] < st["n_coarse"] // 2
    xa = np.concatenate([o["x"] for o in dense])
    xb = np.concatenate([o["x"] for o in dis])
    assert np.linalg.norm(xb - xa) <= 1e-10 * np.linalg.norm(xa)


@pytest.mark.parametrize("name,blocks", [("c2", None), ("c5", None), ("c5", 4)])
def test_full_size_eight_ranks_vs_oracle_golden(name, blocks):
    """SURVEY f1 / §8(e) at full size: config 2 (64 subdomains) and config 5 (the bench workload,
    512 subdomains, 954,947 DOFs) split over 8 loopback ranks in 2x2x2 boxes, coarse problem by
    rank-level dissection (the default for R > 1), against the stored whole-vector oracle solve
    (tests/golden, oracle/ only): velocity and pressure blocks at relative L2 <= 1e-8, iterations
    +-1, kappa 1 %."""
    import torch
    import paper_2304_09770_b200 as vb
    from synthetic.configs import C5_DIMS
    from test_gpu_vem import load_golden
    prob = make_problem(name, dims=C5_DIMS[1]) if name == "c5" else make_problem(name)
    z, meta = load_golden(name)
    ctx1 = vb.context_for(prob)
    ids1 = ctx1.dof_layout()   # 1-rank free order = the golden's order (setup only)
    ctx1.close()
    pos = np.full(int(ids1.max()) + 1, -1, np.int64)
    pos[ids1] = np.arange(ids1.size)
    outs = _run_ranks(prob, (2, 2, 2), check_operator=False, blocks=blocks)
    x = np.full(ids1.size, np.nan)
    for o in outs:
        x[pos[o["ids"]]] = o["x"]
        assert o["stats"]["n_coarse_root"] < o["stats"]["n_coarse"]
        assert abs(o["rep"]["iterations"] - meta["iterations"]) <= 1
        assert abs(o["rep"]["kappa"] - meta["kappa"]) <= 0.01 * meta["kappa"]
    nv = meta["n_free_vel"]
    xo = z["x_full"]
    du = np.linalg.norm(x[:nv] - xo[:nv]) / np.linalg.norm(xo[:nv])
    dp = np.linalg.norm(x[nv:] - xo[nv:]) / np.linalg.norm(xo[nv:])
    print("%s 8 ranks (blocks %s): du %.2e dp %.2e it %d (oracle %d), root %d of N_c %d, local %s"
          % (name, blocks, du, dp, outs[0]["rep"]["iterations"], meta["iterations"], outs[0]["stats"]["n_coarse_root"],
             outs[0]["stats"]["n_coarse"], [o["stats"]["n_coarse_local"] for o in outs]))
    assert du <= 1e-8 and dp <= 1e-8, (du, dp)
