#!/usr/bin/env python
"""Benchmark of the IgA curl-div hot path on B200 (BASELINE.json metric).

A step = one whole PCG + V-cycle solve to rel. residual 1e-8 of a seeded right-hand side
on the workload config (default: BASELINE configs[4], 3D p=4 n=160, the largest single-GPU
config; inputs already resident in HBM).  value = solved DOF/s over all ranks
(ndof * ranks / time-to-solution).  Beside it: operator-apply throughput (L2-flushed by a
rotating buffer set larger than L2), the roofline of the apply kernel measured live inside
the timed solves, the end-to-end number through igacd_solve_host (host buffers), the CPU
oracle on a bounded sample, clocks sampled during the timed region.

  python bench.py [--gpus N] [--steps K] [--warmup W] [--config I] [--impl ours|reference]
N > 1: launched by torch.distributed.run; replicas only (independent problems per rank,
no collective on the data path), max-over-ranks timing.
"""
import argparse
import json
import os
import statistics
import subprocess
import sys
import threading
import time

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

import numpy as np  # noqa: E402

import inputs  # noqa: E402

L2_BYTES = 126 * 2 ** 20


def parse():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=3)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--config", type=int, default=4)
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--maxit", type=int, default=20000)
    ap.add_argument("--apply-reps", type=int, default=0,
                    help="standalone applies per level in the sweep (default: 1000 for config 2, as BASELINE "
                         "configs[2] asks, else 20)")
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--no-e2e", action="store_true")
    ap.add_argument("--no-gmres", action="store_true")
    ap.add_argument("--profile-step", action="store_true",
                    help="bracket the first timed step with cudaProfilerStart/Stop (ncu --profile-from-start off)")
    return ap.parse_args()


def peaks():
    try:
        return json.load(open(os.path.join(ROOT, "MEASURED_PEAKS.json"))), "measured"
    except Exception:
        return {"hbm_gbs": 6650.0, "sm_max_mhz": 1965.0}, "fallback"


class Clocks:
    """nvidia-smi sampling of SM clocks and throttle reasons during the timed region."""

    Q = ("clocks.sm,clocks.max.sm,clocks_event_reasons.hw_slowdown,clocks_event_reasons.hw_thermal_slowdown,"
         "clocks_event_reasons.sw_thermal_slowdown,clocks_event_reasons.sw_power_cap")

    def __init__(self, index):
        self.index, self.rows, self.proc = index, [], None

    def __enter__(self):
        try:
            self.proc = subprocess.Popen(["nvidia-smi", "-i", str(self.index), "--query-gpu=" + self.Q,
                                          "--format=csv,noheader,nounits", "-lms", "200"],
                                         stdout=subprocess.PIPE, stderr=subprocess.DEVNULL, text=True)
            self.th = threading.Thread(target=self._read, daemon=True)
            self.th.start()
        except Exception:
            self.proc = None
        return self

    def _read(self):
        for line in self.proc.stdout:
            parts = [p.strip() for p in line.split(",")]
            if len(parts) == 6:
                self.rows.append(parts)

    def __exit__(self, *a):
        if self.proc:
            self.proc.terminate()
            try:
                self.proc.wait(timeout=2)
            except Exception:
                self.proc.kill()

    def summary(self):
        if not self.rows:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["unavailable"]}
        sm = [float(r[0]) for r in self.rows if r[0].replace(".", "").isdigit()]
        mx = [float(r[1]) for r in self.rows if r[1].replace(".", "").isdigit()]
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        reasons = sorted({names[k] for r in self.rows for k in range(4) if r[2 + k].lower() == "active"})
        return {"sm_mhz": statistics.median(sm) if sm else None, "sm_max_mhz": max(mx) if mx else None,
                "reasons": reasons, "samples": len(self.rows)}


_CPU_CACHE = {}


def cpu_sample(cfg):
    """The oracle (as it stands) on a bounded sample of the workload: the same operator
    (degree, nu, beta, lambda, b0) on a reduced mesh.  Like the GPU step, the timed part is
    the PCG + V-cycle solve; the oracle's assembly and Galerkin hierarchy are set up once
    (untimed).  Returns (DOF/s, seconds, description)."""
    from oracle.krylov import pcg
    from oracle.multigrid import AuxPreconditioner
    from oracle.operator import Discretization, form_alfven
    n = 6 if cfg.dim == 3 else 32
    small = cfg.with_(n=n, levels=2)   # two levels: a V-cycle, like the GPU solve (R6 would stop at one)
    if small not in _CPU_CACHE:
        A = Discretization(small.dim, small.p, small.n).assemble(form_alfven(small.nu, small.beta, small.lam, small.b0))
        mode = "add"   # the library default (reading R8')
        _CPU_CACHE[small] = (A, AuxPreconditioner(A, small.dim, small.p, small.n, small.b0, small.levels, mode=mode))
    A, B = _CPU_CACHE[small]
    b = inputs.rhs(small)
    t0 = time.perf_counter()
    _, it, hist = pcg(A, b, B, small.tol, 5000)
    dt = time.perf_counter() - t0
    desc = ("oracle PCG + aux/2-level V-cycle solve (setup untimed) of %s with n=%d (%d DOFs, %d iterations, "
            "rel.res %.1e)" % (cfg.name, n, small.ndof, it, hist[-1]))
    return small.ndof / dt, dt, desc


def cores():
    try:
        return len(os.sched_getaffinity(0))
    except Exception:
        return os.cpu_count()


def run_reference(args, cfg, rank, world):
    if rank != 0:
        return
    for _ in range(args.warmup):
        cpu_sample(cfg)
    vals, secs = [], []
    desc = ""
    for _ in range(args.steps):
        v, dt, desc = cpu_sample(cfg)
        vals.append(v)
        secs.append(dt)
    value = statistics.mean(vals)
    out = {"impl": "reference", "metric": BASE_METRIC, "value": value, "unit": "DOF/s", "n_gpus": args.gpus,
           "steps": args.steps, "warmup": args.warmup, "ms_per_step": 1000 * statistics.mean(secs),
           "higher_is_better": True, "scaling": "weak", "vs_baseline": None, "dtype": "f64",
           "data": "synthetic (seeded RHS)",
           "config": {"workload": cfg.name, "dim": cfg.dim, "p": cfg.p, "n": cfg.n, "ndof": cfg.ndof},
           "cpu_baseline": {"value": value, "unit": "DOF/s", "cores": cores(), "kind": "oracle", "sample": desc},
           "e2e": {"value": value, "unit": "DOF/s", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0}}
    print(json.dumps(out), flush=True)


BASE_METRIC = json.load(open(os.path.join(ROOT, "BASELINE.json")))["metric"]


def rank_rhs(cfg, rank):
    """Replicas: rank r solves its own seeded right-hand side (seed + r)."""
    return inputs.rhs(cfg, seed=cfg.seed + rank)


def max_over_ranks(value, dist, device):
    """Max of a per-rank time over all ranks (the slowest replica sets the job time)."""
    if dist is None:
        return value
    import torch
    t = torch.tensor([value], dtype=torch.float64, device=device)
    dist.all_reduce(t, op=dist.ReduceOp.MAX)
    return float(t.item())


def precond_timing(ig, h, b, stream, reps=10):
    """Warm CUDA-event times of one vector V-cycle and one preconditioner application."""
    import torch
    z = torch.empty_like(b)
    out = {}
    for name, fn in (("vcycle_ms", ig.igacd_vcycle), ("precond_ms", ig.igacd_precond)):
        for _ in range(2):
            fn(h, b, z)
        torch.cuda.synchronize()
        t0, t1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        t0.record(stream)
        for _ in range(reps):
            fn(h, b, z)
        t1.record(stream)
        torch.cuda.synchronize()
        out[name] = t0.elapsed_time(t1) / reps
    return out


def vcycle_bytes(ig, h, cfg):
    """Algorithmic HBM bytes of one vector V-cycle from x = 0 with the T_n^p smoother, one pre-
    and one post-sweep: every kernel reads each input once and writes
    each output once, 8 B per fp64 value.  Per level with N unknowns (coarse level N' = N / 2^d):
      pre-sweep   x = w T^-1 b: one line-solve pass per axis, 16 N each (3D levels whose [m][m]
                  slab fits in shared memory solve axes 1 and 2 in one pass)
      residual    r = b - A x: 24 N;   restriction r -> b': 8 N + 8 N'
      prolongation x += P x': 8 N' + 16 N
      post-sweep  r = b - A x (24 N), T^-1 passes (16 N each, the last one x += w .: 24 N)
    coarsest level: the dense inverse (8 N^2) plus 16 N."""
    L = ig.igacd_num_levels(h)
    tot = 0.0
    for l in range(L):
        N = ig.igacd_ndof(h, l)
        if l == L - 1:
            tot += 8.0 * N * N + 16.0 * N
            break
        Nc = ig.igacd_ndof(h, l + 1)
        passes = ig.igacd_level_tsolve_passes(h, l)
        pre = 16.0 * N * passes
        post = 24.0 * N + 16.0 * N * (passes - 1) + 24.0 * N
        tot += pre + 24.0 * N + 8.0 * N + 8.0 * Nc + 8.0 * Nc + 16.0 * N + post
    return tot


def main():
    args = parse()
    rank = int(os.environ.get("RANK", "0"))
    world = int(os.environ.get("WORLD_SIZE", "1"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    cfg = inputs.config(args.config)
    if args.impl == "reference":
        return run_reference(args, cfg, rank, world)

    import torch
    torch.cuda.set_device(local)
    dist = None
    if world > 1:
        import torch.distributed as dist
        dist.init_process_group("nccl", device_id=torch.device("cuda", local))
    from paper_1805_10058_b200 import igacd as ig

    def barrier():
        if dist is not None:
            dist.barrier()

    stream = torch.cuda.current_stream()
    torch.cuda.synchronize()
    t_setup = time.perf_counter()
    h = ig.igacd_create(cfg.dim, cfg.p, cfg.n, cfg.nu, cfg.beta, cfg.lam, cfg.b0, levels=cfg.levels)
    torch.cuda.synchronize()
    setup_s = time.perf_counter() - t_setup   # assembly, hierarchy, power iterations, coarse inverse
    N = ig.igacd_ndof(h)
    b_host = rank_rhs(cfg, rank)
    b = torch.from_numpy(b_host).cuda()
    x = torch.zeros_like(b)
    pk, pk_src = peaks()

    # ---- warm-up ----------------------------------------------------------------------
    iters = rel = None
    for _ in range(args.warmup):
        iters, rel = ig.igacd_solve(h, b, x, cfg.tol, args.maxit, raise_on_noconv=False)
    torch.cuda.synchronize()

    # ---- timed solves -----------------------------------------------------------------
    ig.igacd_set_profiling(h, True)
    ig.igacd_reset_profile(h)
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    barrier()
    torch.cuda.synchronize()
    with Clocks(local) as clk:
        e0.record(stream)
        its, rels = [], []
        for k in range(args.steps):
            if args.profile_step and k == 0:
                torch.cuda.profiler.start()
            it, rel = ig.igacd_solve(h, b, x, cfg.tol, args.maxit, raise_on_noconv=False)
            if args.profile_step and k == 0:
                torch.cuda.profiler.stop()
            its.append(it)
            rels.append(rel)
        e1.record(stream)
        torch.cuda.synchronize()
    barrier()
    ms = e0.elapsed_time(e1) / args.steps
    launches, apply_launches, apply_ms = ig.igacd_get_profile(h)
    ig.igacd_set_profiling(h, False)
    ms = max_over_ranks(ms, dist, "cuda")
    value = N * world / (ms / 1000.0)
    converged = all(r < cfg.tol for r in rels)
    # self-check of the timed solves: the TRUE relative residual ||b - A x|| / ||b|| of the last
    # solution (the library's residual kernel; PAPER.md:1333 criterion), not the recursive one
    rv = torch.empty_like(b)
    ig.igacd_residual(h, 0, b, x, rv)
    true_relres = float(torch.linalg.norm(rv)) / float(torch.linalg.norm(b))
    del rv

    # roofline of the dominant kernel (level-0 operator apply inside the timed solves)
    apply_avg_ms = apply_ms / max(apply_launches, 1)
    alg_bytes = 2 * 8 * N            # read x once, write A x once (fp64)
    achieved = alg_bytes / (apply_avg_ms * 1e-3) / 1e9
    traffic = None
    tpath = os.path.join(ROOT, "profiles", "apply_traffic.json")
    if os.path.exists(tpath):
        traffic = json.load(open(tpath)).get(cfg.name)

    # the apply is FP64-issue-bound: algorithmic FP64
    # instructions per unknown of the sum-factorised operator with symmetric pairing,
    # 3D: (66p + 90)/3, 2D: (22p + 26)/2; peak = measured DFMA issue rate
    fp64_per_unknown = (66 * cfg.p + 90) / 3.0 if cfg.dim == 3 else (22 * cfg.p + 26) / 2.0
    fp64_peak = 17.1e12   # tools/microbench/fp64_peak.cu on B200 (59 DFMA/clk/SM at 1.965 GHz)
    fp64_achieved = fp64_per_unknown * N / (apply_avg_ms * 1e-3)

    # ---- GMRES (the paper's PGMRES) on the same system: one solve ---------------------------
    gmres = None
    if not args.no_gmres:
        xg = torch.zeros_like(b)
        g0, g1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        g0.record(stream)
        git, grel = ig.igacd_gmres(h, b, xg, cfg.tol, args.maxit, restart=30, raise_on_noconv=False)
        g1.record(stream)
        torch.cuda.synchronize()
        gmres = {"restart": 30, "iterations": git, "relres": grel,
                 "time_to_solution_s": g0.elapsed_time(g1) / 1000.0}
        del xg

    # ---- one V-cycle and one preconditioner application (CUDA events, warm) --------------
    vc = precond_timing(ig, h, b, stream)
    vc_bytes = vcycle_bytes(ig, h, cfg)
    vc_achieved = vc_bytes / (vc["vcycle_ms"] * 1e-3) / 1e9

    # ---- operator-apply sweep over every level (rotating buffers > L2) ---------------------
    reps = args.apply_reps or (1000 if args.config == 2 else 20)
    sweep = []
    for lvl in range(ig.igacd_num_levels(h)):
        Nl = ig.igacd_ndof(h, lvl)
        nbuf = max(2, int(np.ceil(2 * L2_BYTES / (16 * Nl))) + 1)
        xs = [torch.randn(Nl, dtype=torch.float64, device="cuda") for _ in range(nbuf)]
        ys = [torch.empty(Nl, dtype=torch.float64, device="cuda") for _ in range(nbuf)]
        for k in range(3):
            ig.igacd_apply(h, lvl, xs[k % nbuf], ys[k % nbuf])
        torch.cuda.synchronize()
        a0, a1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        a0.record(stream)
        for k in range(reps):
            ig.igacd_apply(h, lvl, xs[k % nbuf], ys[k % nbuf])
        a1.record(stream)
        torch.cuda.synchronize()
        lms = a0.elapsed_time(a1) / reps
        sweep.append({"level": lvl, "ndof": Nl, "ms": lms, "dof_per_s": Nl / (lms * 1e-3),
                      "gbs": 16 * Nl / (lms * 1e-3) / 1e9, "reps": reps})
        del xs, ys
    sweep_ms = sweep[0]["ms"]

    # ---- end to end through the C ABI with host buffers -----------------------------------
    e2e = None
    if not args.no_e2e:
        bh = torch.from_numpy(b_host).pin_memory()
        xh = torch.empty(N, dtype=torch.float64).pin_memory()
        ig.igacd_solve_host(h, bh, xh, cfg.tol, args.maxit, raise_on_noconv=False)
        barrier()
        torch.cuda.synchronize()
        h0, h1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        h0.record(stream)
        for _ in range(args.steps):
            ig.igacd_solve_host(h, bh, xh, cfg.tol, args.maxit, raise_on_noconv=False)
        h1.record(stream)
        torch.cuda.synchronize()
        ems = h0.elapsed_time(h1) / args.steps
        ems = max_over_ranks(ems, dist, "cuda")
        e2e = {"value": N * world / (ems / 1000.0), "unit": "DOF/s", "h2d_bytes_per_step": 8 * N,
               "d2h_bytes_per_step": 8 * N, "ms_per_step": ems}

    if rank == 0:
        cpu = None
        if world == 1 and not args.no_cpu_baseline:
            v, dt, desc = cpu_sample(cfg)
            cpu = {"value": v, "unit": "DOF/s", "cores": cores(), "kind": "oracle", "sample": desc,
                   "seconds": dt}
        out = {
            "metric": BASE_METRIC, "value": value, "unit": "DOF/s", "n_gpus": world, "steps": args.steps,
            "warmup": args.warmup, "ms_per_step": ms, "higher_is_better": True, "scaling": "weak",
            "vs_baseline": None, "dtype": "f64", "data": "synthetic (seeded RHS, BASELINE config)",
            "config": {"workload": cfg.name, "dim": cfg.dim, "p": cfg.p, "n": cfg.n, "ndof": N,
                       "nu": cfg.nu, "beta": cfg.beta, "lambda": cfg.lam, "b0": list(cfg.b0),
                       "levels": ig.igacd_num_levels(h), "tol": cfg.tol,
                       "l2": "solve vectors exceed L2 (3D) / apply sweep rotates buffer pairs > 2xL2 per level",
                       "parallelism": "replicas" if world > 1 else "single"},
            "time_to_solution_s": ms / 1000.0, "pcg_iterations": its[-1], "relres": rel,
            "converged": converged, "true_relres": true_relres, "setup_s": setup_s,
            "preconditioner": "aux-additive (R8') + V-cycle (Toeplitz smoother R4')",
            "apply": {"dof_per_s": N / (sweep_ms * 1e-3), "ms": sweep_ms,
                      "gbs": 16 * N / (sweep_ms * 1e-3) / 1e9,
                      "hbm_frac": 16 * N / (sweep_ms * 1e-3) / 1e9 / pk["hbm_gbs"]},
            "roofline": {"bound": "hbm", "achieved": achieved, "peak": pk["hbm_gbs"], "unit": "GB/s",
                         "frac": achieved / pk["hbm_gbs"], "traffic": traffic, "peak_source": pk_src,
                         "kernel": ("k_march3d<p=%d> (level-0 apply inside PCG)" % cfg.p if cfg.dim == 3
                                    else "k_op2d<p=%d> (level-0 apply inside PCG)" % cfg.p),
                         "launches": apply_launches, "avg_ms": apply_avg_ms},
            "roofline_fp64": {"bound": "alu", "achieved": fp64_achieved / 1e12, "peak": fp64_peak / 1e12,
                              "unit": "T FP64 instr/s", "frac": fp64_achieved / fp64_peak,
                              "per_unknown": fp64_per_unknown, "peak_source": "measured (tools/microbench)"},
            "apply_sweep": sweep,
            "vcycle": {"ms": vc["vcycle_ms"], "precond_ms": vc["precond_ms"], "bound": "hbm",
                       "achieved": vc_achieved, "peak": pk["hbm_gbs"], "unit": "GB/s",
                       "frac": vc_achieved / pk["hbm_gbs"], "alg_bytes": vc_bytes,
                       "what": "one vector V-cycle (igacd_vcycle) from x = 0; algorithmic bytes per DESIGN.md "
                               "'V-cycle bytes' (each kernel reads its inputs and writes its outputs once)"},
            "gmres": gmres,
            "gpu_launches": launches,
            "clocks": clk.summary(),
            "cpu_baseline": cpu,
            "e2e": e2e,
        }
        print(json.dumps(out), flush=True)
    ig.igacd_destroy(h)
    if dist is not None:
        dist.destroy_process_group()


if __name__ == "__main__":
    main()
