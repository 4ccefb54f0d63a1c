#!/usr/bin/env python
"""Benchmark: PCG+BDDC solve of the divergence-free VEM Stokes system (BASELINE.json metric).

A step = one vb_pcg_solve (rhs condensation B0, the whole PCG loop B1-B7 with the BDDC
preconditioner, back-substitution B8) on the config-5 workload: 32^3 hexahedra (k=2) in 8^3
subdomains of 4^3 cells per GPU, manufactured solution, vertex+edge+face constraints, deluxe
scaling, fp64, rtol 1e-10, x0 = 0.  value = DOF*iterations/s (nDofs in the paper's T2-T4
convention x PCG iterations / T_solve), summed over ranks.

  python bench.py [--gpus N --steps K --warmup W] [--impl reference]
"""
import argparse
import json
import os
import subprocess
import sys
import threading
import time

import numpy as np

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

METRIC = "PCG+BDDC solve time & DOF·iters/s (FP64) at 1/2/4/8 B200; % roofline"
UNIT = "DOF*it/s"


def _peaks():
    try:
        with open(os.path.join(ROOT, "MEASURED_PEAKS.json")) as f:
            p = json.load(f)
        return float(p["hbm_gbs"]), "measured"
    except Exception:
        return 6650.0, "fallback"


def _ncu_traffic(role_key="S_T packed GEMV"):
    """DRAM bytes (read + write) per launch of the dominant kernel from the newest committed
    ncu --set full capture that contains it (profiles/r*_ncu_full_*.json entries carry a "role"),
    or None."""
    import glob
    files = sorted(glob.glob(os.path.join(ROOT, "profiles", "r*_ncu_full_*.json")), reverse=True)
    scale = {"byte": 1.0, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9}
    for path in files:
        try:
            for d in json.load(open(path)):
                if role_key in d.get("role", ""):
                    tot = 0.0
                    for k in ("dram__bytes_read.sum", "dram__bytes_write.sum"):
                        v, u = d[k].split()
                        tot += float(v) * scale[u]
                    return tot, os.path.basename(path)
        except Exception:
            continue
    return None, None


class Clocks:
    """nvidia-smi clocks/throttle sampling during the timed region (B200_PROFILING.md)."""

    def __init__(self, device):
        self.device, self.samples, self.proc = device, [], None

    def __enter__(self):
        q = ("clocks.sm,clocks.max.sm,clocks_event_reasons.hw_slowdown,clocks_event_reasons.hw_thermal_slowdown,"
             "clocks_event_reasons.sw_thermal_slowdown,clocks_event_reasons.sw_power_cap")
        try:
            self.proc = subprocess.Popen(["nvidia-smi", "-i", str(self.device), "--query-gpu=" + q,
                                          "--format=csv,noheader,nounits", "-lms", "100"],
                                         stdout=subprocess.PIPE, stderr=subprocess.DEVNULL, text=True)
            self.t = threading.Thread(target=self._read, daemon=True)
            self.t.start()
        except Exception:
            self.proc = None
        return self

    def _read(self):
        for line in self.proc.stdout:
            parts = [x.strip() for x in line.split(",")]
            if len(parts) == 6:
                self.samples.append(parts)

    def __exit__(self, *a):
        if self.proc:
            time.sleep(0.25)
            self.proc.terminate()
            try:
                self.proc.wait(2)
            except Exception:
                pass

    def summary(self):
        if not self.samples:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["unsampled"]}
        sm = [float(s[0]) for s in self.samples if s[0].replace(".", "").isdigit()]
        mx = [float(s[1]) for s in self.samples if s[1].replace(".", "").isdigit()]
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        reasons = sorted({names[i] for s in self.samples for i in range(4) if s[2 + i].lower() == "active"})
        return {"sm_mhz": float(np.median(sm)) if sm else None, "sm_max_mhz": max(mx) if mx else None,
                "reasons": reasons, "samples": len(self.samples)}


def _dist():
    ws = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    return ws, rank, local


def run_oracle_sample(steps, warmup):
    """The oracle (oracle/, plain NumPy/SciPy) on a bounded sample of the workload: the same 4^3-cell
    subdomains, k=2, constraints and rtol, on a 4^3 subdomain grid (config 2) instead of 8^3."""
    from synthetic import make_problem
    from oracle.assemble import GlobalSystem
    from oracle.bddc import BDDC
    prob = make_problem("c2")
    gs = GlobalSystem(prob)
    bd = BDDC(gs)
    ndofs = gs.dofs.n_dofs_paper()
    for _ in range(warmup):
        bd.solve(rtol=1e-10)
    ts, its = [], []
    for _ in range(steps):
        t0 = time.perf_counter()
        _, _, rep = bd.solve(rtol=1e-10)
        ts.append(time.perf_counter() - t0)
        its.append(rep["iterations"])
    t = float(np.mean(ts))
    return dict(value=ndofs * float(np.mean(its)) / t, t=t, it=float(np.mean(its)), ndofs=ndofs,
                cores=_blas_threads(),
                sample="c5 sampled as c2: the oracle BDDC-PCG solve (B0+PCG+B8, setup excluded) on 64 of "
                       "c5's 512 subdomains (16^3 cells, 4^3 subdomains of 4^3 cells: the same subdomain "
                       "size, k, constraints and rtol; the oracle's per-iteration work is per subdomain, so "
                       "DOF*it/s of the sample stands for c5; the oracle's c5 setup alone takes ~18 min), "
                       "mean of %d solves" % steps)


def _blas_threads():
    """Threads the oracle's BLAS actually uses (threadpoolctl), else the host's core count."""
    try:
        from threadpoolctl import threadpool_info
        n = [d.get("num_threads") for d in threadpool_info() if d.get("user_api") == "blas"]
        if n and n[0]:
            return int(n[0])
    except Exception:
        pass
    return os.cpu_count()


def reference_arm(args):
    ws, rank, _ = _dist()
    if ws > 1 and rank != 0:
        return
    r = run_oracle_sample(args.steps, args.warmup)
    cpu = {"value": r["value"], "unit": UNIT, "cores": r["cores"], "kind": "oracle", "sample": r["sample"]}
    line = {"impl": "reference", "metric": METRIC, "value": r["value"], "unit": UNIT, "n_gpus": args.gpus,
            "steps": args.steps, "warmup": args.warmup, "ms_per_step": r["t"] * 1e3, "higher_is_better": True,
            "scaling": "weak", "vs_baseline": None, "dtype": "f64", "data": "synthetic",
            "config": {"workload": "c5, sampled as c2 (64 of its 512 subdomains; see cpu_baseline.sample)",
                       "iterations": r["it"],
                       "n_dofs": r["ndofs"]},
            "cpu_baseline": cpu,
            "e2e": {"value": r["value"], "unit": UNIT, "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0}}
    print(json.dumps(line))


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=5)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--config", default="c5")
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--no-kernel-timing", action="store_true", help="skip the per-kernel CUDA events")
    ap.add_argument("--coarse-dissection", type=int, default=-1, choices=[-1, 0, 1],
                    help="coarse problem by dissection (1), dense replicated (0), auto (-1)")
    ap.add_argument("--neumann", action="store_true",
                    help="the paper's setting (P:1197): Neumann faces x = 1, y = 1 (DESIGN A35); not the default")
    ap.add_argument("--coarse-blocks", type=int, default=-1,
                    help="parts of the coarse dissection on one GPU (blocks of subdomains; -1 auto)")
    args = ap.parse_args()
    args.warmup = max(args.warmup, 3)
    if args.impl == "reference":
        return reference_arm(args)

    import torch
    ws, rank, local = _dist()
    if ws > 1:
        import torch.distributed as dist
        os.environ.setdefault("MASTER_ADDR", "127.0.0.1")
        # NCCL's communicator lines (rank counts, NVLS/P2P transports) on stderr for the run record
        os.environ.setdefault("NCCL_DEBUG", "INFO")
        os.environ.setdefault("NCCL_DEBUG_SUBSYS", "INIT")
        torch.cuda.set_device(local)
        dist.init_process_group("nccl", device_id=torch.device("cuda", local))
    torch.cuda.set_device(local)
    os.environ["VB_KERNEL_TIMING"] = "0"
    import paper_2304_09770_b200 as vb
    from synthetic import make_problem
    from synthetic.configs import C5_DIMS

    # weak scaling: 32^3 cells per GPU; GPU box layouts 1x1x1 / 1x1x2 / 1x2x2 / 2x2x2
    rank_grid = {1: (1, 1, 1), 2: (1, 1, 2), 4: (1, 2, 2), 8: (2, 2, 2)}.get(ws)
    if ws > 1 and (args.config != "c5" or rank_grid is None):
        raise SystemExit("multi-GPU runs use config c5 on 1, 2, 4 or 8 GPUs")
    dims = C5_DIMS[ws] if args.config == "c5" else None
    prob = make_problem(args.config, dims=dims, neumann=("x1", "y1") if args.neumann else None)
    stream = torch.cuda.current_stream()
    dist_kw = {}
    if ws > 1:
        uid = [vb.nccl_unique_id() if rank == 0 else None]
        torch.distributed.broadcast_object_list(uid, src=0)
        dist_kw = dict(rank=rank, nranks=ws, device=local, nccl_id=uid[0],
                       subdomain_rank=vb.box_ranks(prob.sub_grid, rank_grid))
    t0 = time.perf_counter()
    ctx = vb.context_for(prob, stream=stream, **dist_kw)
    t_setup = time.perf_counter() - t0
    ctx.set_option("coarse_dissection", args.coarse_dissection)
    ctx.set_option("coarse_blocks", args.coarse_blocks)
    t0 = time.perf_counter()
    ctx.factor()
    t_factor = time.perf_counter() - t0
    st = ctx.stats()
    # the same factorisation again on the same context (workspace pages already mapped once in this
    # process): separates the DMMA work from first-touch allocation cost
    t0 = time.perf_counter()
    ctx.factor()
    t_factor_warm = time.perf_counter() - t0
    st_warm = ctx.stats()
    # a third factorisation with CUDA events around every DMMA GEMM launch set: the GEMM kernels'
    # own time (the factor's dominant kernel; its DMMA roofline), not reported as the factor time
    gemm_s = None
    if not args.no_kernel_timing:
        os.environ["VB_KERNEL_TIMING"] = "1"
        ctx.factor()
        os.environ["VB_KERNEL_TIMING"] = "0"
        gemm_s = ctx.stats()["factor_gemm_us"] / 1e6 or None
    rhs = torch.zeros(ctx.n_free, dtype=torch.float64, device="cuda")
    ctx.build_rhs(vb.problem_args(prob), rhs)
    x = torch.zeros_like(rhs)
    for _ in range(args.warmup):
        rep = ctx.pcg_solve(rhs, x, rtol=1e-10)

    def barrier():
        if ws > 1:
            torch.distributed.barrier()

    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    its, ktimes = [], []
    # timed pass: the product path (iterations as one CUDA-graph launch, no per-kernel events)
    os.environ["VB_KERNEL_TIMING"] = "0"
    ctx.pcg_solve(rhs, x, rtol=1e-10)
    with Clocks(local) as clk:
        barrier()
        torch.cuda.synchronize()
        e0.record(stream)
        for _ in range(args.steps):
            rep = ctx.pcg_solve(rhs, x, rtol=1e-10)
            its.append(rep["iterations"])
        e1.record(stream)
        torch.cuda.synchronize()
        barrier()
    ms = e0.elapsed_time(e1) / args.steps
    if ws > 1:
        t = torch.tensor([ms], device="cuda")
        torch.distributed.all_reduce(t, op=torch.distributed.ReduceOp.MAX)
        ms = float(t.item())
    # second timed pass for the roofline: the same solves with CUDA events around every launch of
    # the GEMV categories on the library stream (host-driven iterations: event records are not
    # allowed inside the conditional graph body)
    ms_instr = None
    if not args.no_kernel_timing:
        os.environ["VB_KERNEL_TIMING"] = "1"
        ctx.pcg_solve(rhs, x, rtol=1e-10)
        barrier()
        torch.cuda.synchronize()
        e0.record(stream)
        for _ in range(args.steps):
            ctx.pcg_solve(rhs, x, rtol=1e-10)
            ktimes.append(ctx.kernel_times())
        e1.record(stream)
        torch.cuda.synchronize()
        barrier()
        ms_instr = e0.elapsed_time(e1) / args.steps
        os.environ["VB_KERNEL_TIMING"] = "0"
    # K7, the element-by-element saddle operator (north-star subsystem 3; not in the solve, which applies
    # the explicit interface Schur complement): device time of elem_apply per launch (CUDA events on the
    # library stream), algorithmic bytes 8 sum_K (nv (nv + 1) / 2 + np nv) (SURVEY §8(d) b_e)
    k7_ms = None
    if not args.no_kernel_timing:
        os.environ["VB_KERNEL_TIMING"] = "1"
        y = torch.empty_like(rhs)
        ctx.apply_operator(x, y)
        k7 = []
        for _ in range(max(3, args.steps)):
            ctx.apply_operator(x, y)
            k7.append(ctx.kernel_times().get("elem_apply K7 (packed element matrices)", float("nan")))
        k7_ms = float(np.mean(k7))
        os.environ["VB_KERNEL_TIMING"] = "0"
    it = float(np.mean(its))
    ndofs = st["n_dofs_paper"]          # the whole (global) problem, all ranks together
    value = ndofs * it / (ms / 1e3)

    # e2e: the public API with HOST buffers (pinned), H2D of the rhs and D2H of x inside the call
    rhs_h = torch.empty(ctx.n_free, dtype=torch.float64, pin_memory=True)
    rhs_h.copy_(rhs.cpu())
    x_h = torch.empty(ctx.n_free, dtype=torch.float64, pin_memory=True)
    rn, xn = rhs_h.numpy(), x_h.numpy()
    ctx.pcg_solve_host(rn, xn)
    torch.cuda.synchronize()
    e2 = time.perf_counter()
    e2e_its = []
    for _ in range(args.steps):
        r2 = ctx.pcg_solve_host(rn, xn)
        e2e_its.append(r2["iterations"])
    e2e_ms = (time.perf_counter() - e2) * 1e3 / args.steps
    if ws > 1:
        t = torch.tensor([e2e_ms], device="cuda")
        torch.distributed.all_reduce(t, op=torch.distributed.ReduceOp.MAX)
        e2e_ms = float(t.item())
    e2e_val = ndofs * float(np.mean(e2e_its)) / (e2e_ms / 1e3)

    # roofline of the dominant kernel (the packed symmetric GEMV on S_T)
    if not ktimes or not ktimes[0]:
        ktimes = [{n: float("nan") for n in ("op", "loc", "coarse", "S", "M")}]
    kt = {k: float(np.mean([d[k] for d in ktimes])) for k in ktimes[0]}
    peak, peak_src = _peaks()
    names = list(kt.keys())
    op_ms = kt[names[0]]
    op_bytes = 8.0 * st["sum_pk_G"]
    loc_ms, loc_bytes = kt[names[1]], 8.0 * st["sum_pk_D"]
    c_ms, c_bytes = kt[names[2]], 8.0 * st["pk_coarse"]
    achieved = op_bytes / (op_ms / 1e3) / 1e9
    # the committed ncu capture is of the c5 one-GPU workload: no traffic figure for other configs
    traffic, traffic_src = _ncu_traffic() if (args.config == "c5" and ws == 1 and not args.neumann) else (None, None)
    npr = {2: 4, 3: 10, 4: 20}[prob.k]
    k7_bytes = 8.0 * st["n_cells"] * (st["nv_max"] * (st["nv_max"] + 1) / 2 + npr * st["nv_max"])
    k7_entry = {"ms": k7_ms, "bytes_per_launch": k7_bytes,
                "GBps": k7_bytes / (k7_ms / 1e3) / 1e9 if k7_ms else None,
                "frac": k7_bytes / (k7_ms / 1e3) / 1e9 / peak if k7_ms else None,
                "bytes_note": "every cell counted with nv = nv_max (exact for hexahedral cells)"}
    iter_ms = ms / max(it, 1)
    per_iter_bytes = st["bytes_per_iter"]
    line = {
        "metric": METRIC, "value": value, "unit": UNIT, "n_gpus": ws, "steps": args.steps, "warmup": args.warmup,
        "ms_per_step": ms, "higher_is_better": True, "scaling": "weak", "vs_baseline": None, "dtype": "f64",
        "data": "synthetic",
        "config": {"workload": "%s: %dx%dx%d hex cells, k=%d, %d subdomains%s"
                               % ((args.config,) + tuple(prob.mesh.dims) + (prob.k, int(prob.cell_subdomain.max()) + 1,
                                  (" of 4^3 cells (32^3 cells per GPU)" if args.config == "c5" else "")
                                  + (", Neumann faces x=1, y=1" if args.neumann else ""))),
                   "n_dofs": ndofs, "iterations": it, "kappa": rep["kappa"], "rel_residual": rep["rel_residual"],
                   "n_primal": st["n_primal"], "n_coarse": st["n_coarse"], "rtol": 1e-10,
                   "coarse": ("dissection: root %d, local %d" % (st["n_coarse_root"], st["n_coarse_local"])
                              if st["n_coarse_root"] else "dense replicated inverse"),
                   "t_setup_s": t_setup, "t_factor_s": t_factor,
                   "parallelism": "subdomains on 1 GPU" if ws == 1 else
                   "subdomain boxes on %d GPUs (rank grid %s), NCCL interface exchange / coarse gather / dots"
                   % (ws, "x".join(map(str, rank_grid))),
                   "l2": "inputs larger than L2 (%.1f GB of operators streamed per iteration)" % (per_iter_bytes / 1e9),
                   "ms_per_iteration": iter_ms,
                   "ms_per_step_instrumented": ms_instr,
                   "iteration_driver": "CUDA graph, conditional WHILE node (device-side stopping test)",
                   "achieved_GBps_per_iteration_model": per_iter_bytes / (iter_ms / 1e3) / 1e9},
        "roofline": {"bound": "hbm", "kernel": names[0], "measured_in": "second timed pass (per-launch CUDA events)", "achieved": achieved, "peak": peak, "unit": "GB/s",
                     "frac": achieved / peak, "traffic": traffic, "traffic_source": traffic_src,
                     "peak_source": peak_src,
                     "bytes_per_launch": op_bytes, "ms_per_launch": op_ms,
                     "others": {names[1]: {"ms": loc_ms, "GBps": loc_bytes / (loc_ms / 1e3) / 1e9 if loc_ms else None},
                                names[2]: {"ms": c_ms, "GBps": c_bytes / (c_ms / 1e3) / 1e9 if c_ms else None},
                                names[3]: {"ms": kt[names[3]]}, names[4]: {"ms": kt[names[4]]},
                                "elem_apply K7 (element-by-element operator, packed A^K)": k7_entry}},
        "factor": {"t_s": t_factor, "dmma_gemm_flops": st["factor_gemm_flops"],
                   "tflops": st["factor_gemm_flops"] / t_factor / 1e12,
                   "frac_of_dmma_peak": st["factor_gemm_flops"] / t_factor / 37.2e12,
                   "alloc_s": st["factor_alloc_us"] / 1e6,
                   "tflops_excl_alloc": st["factor_gemm_flops"] / max(t_factor - st["factor_alloc_us"] / 1e6, 1e-9) / 1e12,
                   "t_warm_s": t_factor_warm, "alloc_warm_s": st_warm["factor_alloc_us"] / 1e6,
                   "tflops_warm": st["factor_gemm_flops"] / t_factor_warm / 1e12,
                   "frac_of_dmma_peak_warm": st["factor_gemm_flops"] / t_factor_warm / 37.2e12,
                   "gemm_kernel_s": gemm_s,
                   "gemm_kernel_tflops": st["factor_gemm_flops"] / gemm_s / 1e12 if gemm_s else None,
                   "gemm_kernel_frac_of_dmma_peak": st["factor_gemm_flops"] / gemm_s / 37.2e12 if gemm_s else None,
                   "peak_note": "DMMA 37.2 TFLOP/s measured by tools/fp64_peak.cu (profiles/r01_fp64_peak.txt); "
                                "t_s includes the non-GEMM kernels, host work and device allocation (alloc_s: "
                                "first-touch mapping of the factor workspace, varies run to run) of vb_factor; "
                                "*_warm: a second vb_factor on the same context"},
        "e2e": {"value": e2e_val, "unit": UNIT, "h2d_bytes_per_step": 8 * ctx.n_free,
                "d2h_bytes_per_step": 8 * ctx.n_free, "ms_per_step": e2e_ms},
        # kernels per solve (single rank): 24 + 21 it with the coarse dissection, 24 + 15 it with the
        # dense coarse inverse, counted in the ncu launch lists of host-driven c5 solves
        # (profiles/r02t_, r02k_launches_c5_solve_hostdriven_summary.txt; the graph runs the same
        # kernels); multi-rank runs add the exchange pack/sum kernels (not counted here)
        "gpu_launches": int(args.steps * (24 + (21 if st["n_coarse_root"] else 15) * it)),
        "clocks": clk.summary(),
    }
    if rank == 0 and ws == 1 and not args.no_cpu_baseline:
        r = run_oracle_sample(1, 0)
        line["cpu_baseline"] = {"value": r["value"], "unit": UNIT, "cores": r["cores"], "kind": "oracle",
                                "sample": r["sample"]}
    if rank == 0:
        print(json.dumps(line))
    ctx.close()
    if ws > 1:
        torch.distributed.destroy_process_group()


if __name__ == "__main__":
    main()
