#!/usr/bin/env python3
"""bench.py -- PCG-MSP solve throughput on B200 (BASELINE.json metric).

    python bench.py [--gpus N] [--steps K] [--warmup W] [--impl ours|reference]
                    [--config 1] [--precond msp] [--mu 0.8] [--rtol 1e-8]

A *step* is one complete PCG solve L_G x = b to rtol 1e-8 (x0 = 0) with the
MSP preconditioner R = P(mu) L_T~^+ P(mu)^T.  The default workload is the
largest single-GPU configuration that the metric names no size for:
BASELINE configs[2] (3D 7-point anisotropic grid 256^3, 16.8M vertices,
weights 1 (x, y) / 1e-3 (z) x uniform[0.9, 1.1], b ~ N(0,1) projected off
ones); --config 1 / 3 give the 2D 1024^2 grid and the 4M-point random
geometric graph.  value = nnz(L_G) x iterations x (ranks) / seconds.
Setup (GPU hierarchy + expansion + MSP) is timed separately (setup_ms).

Multi-GPU (torchrun, N > 1): the ranks solve ONE system together through
msp_dist_solve (row partition, NCCL halo exchange / all-reduces / all-gather
inside the library) -> "scaling": "strong"; timing is the max over ranks.
--replicas gives the old one-problem-per-rank mode ("weak"); --dist runs the
partitioned path at N = 1 too.

--impl reference times the oracle (oracle/, plain fp64 CPU, test
infrastructure) on the host cores on a bounded sample of the same workload.
"""
from __future__ import annotations

import argparse
import json
import os
import statistics
import subprocess
import sys
import time

import numpy as np

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

METRIC = "PCG-MSP solve nnz*iters/s"
UNIT = "nnz*iters/s"


def env_int(k, d):
    try:
        return int(os.environ.get(k, d))
    except ValueError:
        return d


def measured_peaks():
    try:
        with open(os.path.join(ROOT, "MEASURED_PEAKS.json")) as f:
            p = json.load(f)
        return float(p["hbm_gbs"]), "measured (MEASURED_PEAKS.json hbm_gbs)"
    except Exception:
        return 6650.0, "fallback (B200_PROFILING.md 6.65 TB/s)"


class ClockSampler:
    """nvidia-smi clocks / throttle reasons during the timed region."""

    QUERY = ("index,clocks.sm,clocks.max.sm,power.draw,clocks_event_reasons.active,"
             "clocks_event_reasons.hw_slowdown,clocks_event_reasons.hw_thermal_slowdown,"
             "clocks_event_reasons.sw_thermal_slowdown,clocks_event_reasons.sw_power_cap")

    def __init__(self, gpu_index: int):
        self.idx = gpu_index
        self.proc = None
        self.path = f"/tmp/bench_clocks_{os.getpid()}.csv"

    def start(self):
        try:
            self.proc = subprocess.Popen(
                ["nvidia-smi", f"--id={self.idx}", f"--query-gpu={self.QUERY}", "--format=csv,noheader,nounits",
                 "-lms", "100"], stdout=open(self.path, "w"), stderr=subprocess.DEVNULL)
        except Exception:
            self.proc = None

    def stop(self) -> dict:
        if self.proc is None:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["nvidia-smi unavailable"]}
        self.proc.terminate()
        try:
            self.proc.wait(timeout=5)
        except Exception:
            self.proc.kill()
        sm, smax, reasons = [], [], set()
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        try:
            for line in open(self.path):
                f = [x.strip() for x in line.split(",")]
                if len(f) < 9:
                    continue
                try:
                    sm.append(float(f[1])); smax.append(float(f[2]))
                except ValueError:
                    continue
                for nm, v in zip(names, f[5:9]):
                    if v.lower().startswith("active"):
                        reasons.add(nm)
        except FileNotFoundError:
            pass
        return {"sm_mhz": statistics.median(sm) if sm else None,
                "sm_max_mhz": max(smax) if smax else None,
                "samples": len(sm), "reasons": sorted(reasons)}


# ------------------------------------------------------------ byte models
# Algorithmic HBM bytes per launch: every array the
# kernel must touch, once; gathered neighbour values are L2 re-reads and are
# not counted.
def spmv_bytes(n: int, nnz_adj: int) -> int:
    """p = z + beta p_old fused with q = L_G p, (p, q) and the deferred
    x += alpha p_old: per row the (z_i, p_old_i) pair read, p_i and q_i
    written, x_i read and written (48 B); per adjacency entry an int32 column
    and an fp64 weight (12 B).  SELL padding and gathered neighbour pairs
    (L2 re-reads) are not counted."""
    return n * 48 + nnz_adj * 12


def tile_up_bytes(sizes, kt: int) -> int:
    """r -= a q, (r, r), (r, H): r, q, H read and r written (32 B per
    level-1 node); descendant offsets of the level-Kt nodes (4 B) and y
    written at level Kt (8 B)."""
    n = sizes[0]
    return 32 * n + 12 * sizes[kt - 1]


def tile_down_bytes(sizes, kt: int) -> int:
    """r read and R r written (16 B per level-1 node); the packed factors:
    K'^{-1} of every aggregate at levels 2..Kt (24 B each) and the
    coefficients of the leftovers among levels 1..Kt-1 (24 B each, n_k -
    2 n_{k+1} of them); child pointers of levels 2..Kt (4 B); z, w read at
    level Kt (16 B).  Subtree sizes are recomputed in shared memory."""
    n = sizes[0]
    leftovers = sum(sizes[k] - 2 * sizes[k + 1] for k in range(kt - 1))
    return (16 * n + 24 * sum(sizes[1:kt]) + 24 * leftovers + 4 * sum(sizes[1:kt])
            + 16 * sizes[kt - 1])


# The paper's own counts and timings (context only: Matlab code, FGMRES on the
# expanded system, a 1.1 GHz Intel i7-10710U with 16 GB of RAM, PAPER.md
# l.847-849; unweighted 2D grids, b = [1, ..., 1, 1-n], eps = 1e-8).
PAPER_CONTEXT = {
    "source": "PAPER.md Table 3 (l.859-879), MSP and PEGP, level = max; hardware l.847-849",
    "hardware": "Matlab, Intel i7-10710U @ 1.1 GHz, 16 GB RAM",
    "grid_msp_levelmax": {"n": [256, 1024, 4096, 16384], "steps": [58, 93, 151, 248],
                          "time_s": [0.0133, 0.0793, 0.2281, 1.2778]},
    "grid_pegp_levelmax": {"n": [256, 1024, 4096, 16384], "steps": [7, 6, 5, 4],
                           "time_s": [0.0092, 0.0527, 0.1933, 0.7758]},
    "largest_real_world_msp": {"graph": "tsyl201 (20,685 nodes, 2,454,957 edges)", "mu": 0.8, "steps": 54,
                               "time_s": 3.2941, "eps": 1e-6, "table": "Table 6 (l.976-1001)"},
    "note": "different graphs, sizes, solver (FGMRES) and hardware: not a baseline",
}


# ------------------------------------------------------------ reference arm
# The oracle's own setup scales with the graph (scipy triple products and a
# SuperLU factorisation of L_T~: minutes and tens of GB at configs[2]), so the
# CPU baseline runs it on a bounded sample: the same graph family, weight
# distribution, mu and rhs recipe at a reduced linear size (the metric,
# nnz*iters/s, is per unit of work), one process per host core.
SAMPLE_SCALE = {0: 1.0, 1: 0.25, 2: 0.25, 3: 0.25, 4: 0.05}


class OracleWorkload:
    """The oracle (as it stands) on a bounded sample of the workload; setup
    is untimed."""

    def __init__(self, cfg: int, mu: float, log, precond: str = "msp"):
        from inputs import graphs as G
        from oracle import aggregation as A, expansion as E, graph as GR, precond as PR
        t0 = time.time()
        self.scale = SAMPLE_SCALE.get(cfg, 0.25)
        self.precond = precond
        self.g = G.config_graph(cfg, self.scale)
        h = A.build_hierarchy(self.g, 0)
        if precond == "pegp":
            self.R = PR.pegp(E.expand(self.g, h, mu))
        elif precond == "none":
            self.R = lambda v: v
        else:
            self.R = PR.msp(E.expand_msp_only(self.g, h, mu))
        self.L = GR.laplacian_of_graph(self.g)
        self.b = G.rhs(self.g.n, 0)
        log(f"oracle setup {time.time() - t0:.1f}s (sample: configs[{cfg}] at scale {self.scale}, n={self.g.n})")
        self.one = None

    def describe(self, cfg):
        solver = {"msp": "SuperLU solve of L_T~", "pegp": "SuperLU solve of L_H~", "none": "no preconditioner"}
        return (f"configs[{cfg}] family at linear scale {self.scale} (n={self.g.n}, nnz(L)={self.g.nnz_laplacian}): "
                f"PCG-{self.precond.upper()} iterations of the oracle (scipy SpMV + {solver[self.precond]}), one "
                "process per host core, all on the same sample; oracle setup untimed")

    def _iters(self, iters):
        from oracle import pcg as PC
        L, R = self.L, self.R
        t = time.time()
        res = PC.pcg(lambda v: L @ v, self.b, R, 0.0, iters)
        return res.iterations, time.time() - t

    def sample(self, seconds: float, cores: int = 1):
        """PCG-MSP iterations for about `seconds` on `cores` processes:
        (aggregate nnz*iters/s, total iterations, wall seconds, cores)."""
        if cores <= 1:
            if self.one is None:
                it, dt = self._iters(2)
                self.one = max(dt / 2, 1e-4)
            it, dt = self._iters(max(2, int(seconds / self.one)))
            return self.g.nnz_laplacian * it / dt, it, dt, 1
        import multiprocessing as mp
        global _WL
        _WL = self
        ctx = mp.get_context("fork")          # children share the factorisation
        with ctx.Pool(cores) as pool:
            if self.one is None:               # per-iteration time with every core busy
                t = time.time()
                pool.map(_sample_child, [3] * cores)
                self.one = max((time.time() - t) / 3, 1e-4)
            iters = max(2, int(seconds / self.one))
            t = time.time()
            res = pool.map(_sample_child, [iters] * cores)
            wall = time.time() - t
        tot = sum(r[0] for r in res)
        return self.g.nnz_laplacian * tot / wall, tot, wall, cores


_WL = None


def _sample_child(iters):
    os.environ["OMP_NUM_THREADS"] = "1"
    return _WL._iters(iters)


def host_cores():
    try:
        return len(os.sched_getaffinity(0))
    except Exception:
        return os.cpu_count() or 1


def run_reference(args, rank):
    if rank != 0:
        return 0
    log = lambda m: print(f"[bench/reference] {m}", file=sys.stderr, flush=True)
    wl = OracleWorkload(args.config, args.mu, log, args.precond)
    cores = host_cores()
    per_step = max(2.0, 90.0 / max(1, args.steps + args.warmup))
    vals = []
    for s in range(args.warmup + args.steps):
        v = wl.sample(per_step, cores)
        if s >= args.warmup:
            vals.append(v)
    iters = sum(v[1] for v in vals)
    secs = sum(v[2] for v in vals)
    value = wl.g.nnz_laplacian * iters / secs
    out = {
        "impl": "reference", "metric": METRIC, "value": value, "unit": UNIT, "n_gpus": args.gpus,
        "steps": args.steps, "warmup": args.warmup, "ms_per_step": 1000 * secs / len(vals),
        "higher_is_better": True, "scaling": "strong" if args.gpus > 1 else "weak", "vs_baseline": None,
        "dtype": "f64", "data": "synthetic", "config": config_dict(args, wl.g),
        "cpu_baseline": {"value": value, "unit": UNIT, "cores": cores, "kind": "oracle",
                         "sample": f"{vals[0][1]} iterations per step in total; " + wl.describe(args.config)},
        "e2e": {"value": value, "unit": UNIT, "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
    }
    print(json.dumps(out), flush=True)
    return 0


def config_dict(args, g, extra=None, parallelism=None):
    names = {0: "2D grid 32x32, uniform[1,10] weights", 1: "2D grid 1024x1024, log-uniform[1e-3,1e3] weights",
             2: "3D 7-point anisotropic grid 256^3", 3: "random geometric graph 4M points",
             4: "Chung-Lu power-law 50M vertices (largest component)"}
    d = {"workload": f"BASELINE configs[{args.config}]: {names.get(args.config, '?')}; PCG+{args.precond.upper()} "
                     f"to rtol {args.rtol:g}",
         "n": g.n if g is not None else None, "nnz_L": g.nnz_laplacian if g is not None else None,
         "precond": args.precond, "mu": args.mu, "rtol": args.rtol, "levels": "max",
         "parallelism": parallelism or f"independent problem per rank x{args.gpus}",
         "l2": "flushed (256 MiB write) before every timed step, inside the timed region"}
    if extra:
        d.update(extra)
    return d


class GraphInfo:
    def __init__(self, n, nnz_adj):
        self.n = int(n)
        self.nnz_adj = int(nnz_adj)
        self.nnz_laplacian = self.nnz_adj + self.n


# ------------------------------------------------------------ our arm
def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=3)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--config", type=int, default=2)
    ap.add_argument("--precond", default="msp", choices=["msp", "none", "pegp"])
    ap.add_argument("--inner-rtol", type=float, default=1e-13, help="PEGP: inner CG relative residual (R13)")
    ap.add_argument("--mu", type=float, default=0.8)
    ap.add_argument("--rtol", type=float, default=1e-8)
    ap.add_argument("--maxit", type=int, default=200000)
    ap.add_argument("--dist", action="store_true",
                    help="row-partitioned solve (msp_dist_solve) even at one GPU; the default for N > 1")
    ap.add_argument("--replicas", action="store_true",
                    help="N > 1: one independent problem per rank instead of one partitioned problem")
    ap.add_argument("--no-cpu-baseline", action="store_true")
    args = ap.parse_args()

    rank = env_int("RANK", 0)
    world = env_int("WORLD_SIZE", 1)
    local = env_int("LOCAL_RANK", 0)
    if args.impl == "reference":
        return run_reference(args, rank)

    # stdout carries exactly one JSON line: keep NCCL's banner off it
    os.environ.setdefault("NCCL_DEBUG", "WARN")
    import torch
    import torch.distributed as dist
    from inputs import device as D, graphs as G
    import paper_2207_07847_b200 as M
    from paper_2207_07847_b200 import dist as MD

    log = (lambda m: print(f"[bench r{rank}] {m}", file=sys.stderr, flush=True))
    torch.cuda.set_device(local)
    dev = torch.device("cuda", local)
    if world > 1:
        dist.init_process_group("nccl", device_id=dev)
    use_dist = (world > 1 and not args.replicas) or args.dist
    if use_dist and args.precond != "msp":
        raise SystemExit("the partitioned solve is PCG-MSP")
    if use_dist and world == 1 and not dist.is_initialized():
        import socket
        with socket.socket() as sk:
            sk.bind(("127.0.0.1", 0))
            port = sk.getsockname()[1]
        os.environ.setdefault("MASTER_ADDR", "127.0.0.1")
        os.environ.setdefault("MASTER_PORT", str(port))
        dist.init_process_group("nccl", rank=0, world_size=1, device_id=dev)

    t0 = time.time()
    n, rp, col, val = D.config_csr(args.config, 1.0, 0, dev)
    g = GraphInfo(n, int(rp[-1].item()))
    b_np = G.rhs(g.n, 0)
    log(f"graph n={g.n} nnz(L)={g.nnz_laplacian} in {time.time() - t0:.1f}s")
    t0 = time.time()
    S = M.setup(n, rp, col, val, mu=args.mu, seed=0)
    del rp, col, val
    info = S.info()
    pinfo = None
    if args.precond == "pegp":
        S.pegp_params(args.inner_rtol, 200000, 0)
        pinfo = S.pegp_info()
        log(f"PEGP: H~ nnz {pinfo['hnnz']}, build {pinfo['build_ms']:.1f} ms, coarse level {pinfo['coarse_level']}")
    log(f"setup {info['setup_ms']:.1f} ms (wall {time.time() - t0:.1f}s) levels={info['levels']} "
        f"n~={info['n_tilde']} mwm_rounds={info['mwm_rounds']}")
    drange = None
    if use_dist:
        drange = MD.dist_init(S)
        log(f"partition: rows [{drange[0]}, {drange[1]}) kp={drange[2]} tp={drange[3]} "
            f"halo send={drange[4]} recv={drange[5]}")

    def solve(b_, x_):
        if use_dist:
            return MD.dist_solve(S, b_, x_, rtol=args.rtol, maxit=args.maxit)
        return S.pcg_solve(b_, x_, rtol=args.rtol, maxit=args.maxit, precond=args.precond)

    b = torch.as_tensor(b_np, device=dev)
    x = torch.empty_like(b)
    flush = torch.empty(256 * 1024 * 1024 // 4, dtype=torch.float32, device=dev)
    stream = torch.cuda.current_stream()

    for _ in range(args.warmup):
        flush.fill_(1.0)
        rep = solve(b, x)
    log(f"warmup: {rep['iterations']} iterations, converged={rep['converged']}, "
        f"{rep['solve_ms']:.1f} ms")

    sampler = ClockSampler(local)
    sampler.start()
    time.sleep(0.3)
    if world > 1:
        dist.barrier()
    torch.cuda.synchronize()
    ev0 = torch.cuda.Event(enable_timing=True)
    ev1 = torch.cuda.Event(enable_timing=True)
    ev0.record(stream)
    iters, launches = [], 0
    for _ in range(args.steps):
        flush.fill_(1.0)
        rep = solve(b, x)
        iters.append(rep["iterations"])
        launches += rep["kernel_launches"] + 1
        last_rep = rep
    ev1.record(stream)
    torch.cuda.synchronize()
    if world > 1:
        dist.barrier()
    clocks = sampler.stop()
    ms_total = ev0.elapsed_time(ev1)
    if world > 1:
        t = torch.tensor([ms_total], device=dev, dtype=torch.float64)
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        ms_total = float(t.item())
    ms_step = ms_total / args.steps
    solve_inner = S.pegp_info()["last_solve_inner_iterations"] if args.precond == "pegp" else None
    it = int(np.median(iters))
    # partitioned: all ranks solve ONE system (strong scaling); replicas: one each (weak)
    copies = 1 if use_dist else world
    value = copies * g.nnz_laplacian * sum(iters) / (ms_total / 1000.0)

    # ---- e2e: same metric through the C ABI with host buffers (pinned)
    bh = torch.as_tensor(b_np).pin_memory()
    xh = torch.empty_like(bh).pin_memory()
    solve(bh, xh)
    torch.cuda.synchronize()
    e_iters = []
    if world > 1:
        dist.barrier()
    te = time.perf_counter()
    for _ in range(max(1, min(args.steps, 3))):
        flush.fill_(1.0)
        r2 = solve(bh, xh)
        e_iters.append(r2["iterations"])
    torch.cuda.synchronize()
    te = time.perf_counter() - te
    if world > 1:  # slowest rank
        t = torch.tensor([te], device=dev, dtype=torch.float64)
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        te = float(t.item())
    e2e_value = copies * g.nnz_laplacian * sum(e_iters) / te

    # ---- profiled replay of one step: per-kernel device time (CUDA events
    # bracketing each launch on the solve's stream; serialised, no graph)
    S.set_profiling(True)
    flush.fill_(1.0)
    if args.precond == "pegp":   # one preconditioner apply (the inner CG) stands for the step's kernels
        S.apply_R(b, precond="pegp")
    else:
        solve(b, x)
    S.set_profiling(False)
    prof = S.get_profile()
    sizes = S.level_sizes()
    sz = [int(v) for v in sizes]
    kt = int(info["tile_level"])
    n_own = g.n if not use_dist else int(drange[1] - drange[0])
    nnz_own = g.nnz_adj if not use_dist else int(round(g.nnz_adj * n_own / g.n))
    model = {"spmv": spmv_bytes(n_own, nnz_own)}
    if kt >= 2:  # a generic (per-level) first tier has no tile byte model: its sweeps report time only
        model["tile_up"] = tile_up_bytes(sz, kt)
        model["tile_down"] = tile_down_bytes(sz, kt)
    if use_dist and world > 1:  # the tile byte models are whole-graph figures
        model = {"spmv": model["spmv"]}
    if args.precond == "pegp":
        # k_h_spmv: H~ CSR (12 B per entry) + per row: row pointer 8, row list 4,
        # own (z, p) pair 16, q 8, p 8
        model = {"pegp_spmv": 12 * pinfo["hnnz"] + 44 * int(info["n_tilde"])}
    hbm, peak_src = measured_peaks()
    breakdown = {}
    for k, v in prof.items():
        if v["launches"]:
            avg = v["ms"] / v["launches"]
            e = {"total_ms": round(v["ms"], 3), "launches": v["launches"], "avg_us": round(avg * 1000, 3)}
            if k in model:
                e["GBps"] = round(model[k] / (avg / 1000) / 1e9, 1)
            breakdown[k] = e
    dom = max((k for k in breakdown if k in model), key=lambda k: breakdown[k]["total_ms"])
    ach = model[dom] / (breakdown[dom]["avg_us"] * 1e-6) / 1e9
    traffic = None
    tpath = os.path.join(ROOT, "profiles", "ncu_traffic.json")
    if os.path.exists(tpath):
        try:
            traffic = json.load(open(tpath)).get(f"config{args.config}", {}).get(dom)
        except Exception:
            traffic = None
    roofline = {"bound": "hbm", "kernel": dom, "achieved": round(ach, 1), "peak": hbm, "unit": "GB/s",
                "frac": round(ach / hbm, 4), "traffic": traffic, "peak_source": peak_src,
                "bytes_per_launch": model[dom]}
    prof_total = sum(v["ms"] for v in prof.values())
    solve_bytes = sum(model.get(k, 0) * prof[k]["launches"] for k in prof)
    whole_gbps = solve_bytes / (prof_total / 1000) / 1e9 if prof_total else None

    cpu = None
    if rank == 0 and world == 1 and not args.no_cpu_baseline:
        try:
            wl = OracleWorkload(args.config, args.mu, log, args.precond)
            v, cit, cdt, ncores = wl.sample(15.0, host_cores())
            cpu = {"value": v, "unit": UNIT, "cores": ncores, "kind": "oracle",
                   "sample": f"{cit} iterations in {cdt:.1f}s in total; " + wl.describe(args.config)}
        except Exception as ex:  # reported, never fatal
            cpu = {"value": None, "unit": UNIT, "cores": host_cores(), "kind": "oracle", "sample": f"failed: {ex}"}

    if rank == 0:
        par = (f"row-partitioned x{world} (msp_dist_solve: NCCL halo / all-reduce / all-gather)" if use_dist
               else f"independent problem per rank x{world}")
        extra = {"levels_built": int(info["levels"]), "n_tilde": int(info["n_tilde"]),
                 "tile_level": int(info["tile_level"]), "coarse_level": int(info["coarse_level"]),
                 "ntiles": int(info["ntiles"]), "ntiers": int(info["ntiers"])}
        if pinfo is not None:
            extra["pegp"] = {"inner_iterations_per_solve": solve_inner,"hnnz": pinfo["hnnz"], "build_ms": pinfo["build_ms"], "inner_rtol": args.inner_rtol,
                             "inner_iterations_per_step": S.pegp_info()["last_inner_iterations"],
                             "note": "inner iterations of the profiled apply; kernel_breakdown is that apply"}
        if use_dist:
            extra["partition_level"] = int(drange[2])
            extra["rank0_rows"] = int(drange[1] - drange[0])
            extra["rank0_halo"] = {"send": int(drange[4]), "recv": int(drange[5])}
        out = {
            "metric": METRIC, "value": value, "unit": UNIT, "n_gpus": world, "steps": args.steps,
            "warmup": args.warmup, "ms_per_step": ms_step, "higher_is_better": True,
            "scaling": "strong" if use_dist else "weak",
            "vs_baseline": None, "dtype": "f64", "data": "synthetic",
            "config": config_dict(args, g, extra, par),
            "iterations": it, "converged": bool(last_rep["converged"]), "relres": float(last_rep["relres"]),
            # not converged = the step is `maxit` outer iterations (a bounded sample of the solve)
            "time_to_rtol_s": ms_step / 1000.0 if last_rep["converged"] else None, "setup_ms": info["setup_ms"],
            "solve_GBps_algorithmic": round(whole_gbps, 1) if whole_gbps else None,
            "roofline": roofline, "kernel_breakdown": breakdown,
            "cpu_baseline": cpu,
            "e2e": {"value": e2e_value, "unit": UNIT, "h2d_bytes_per_step": 8 * g.n,
                    "d2h_bytes_per_step": 8 * g.n},
            "gpu_launches": launches, "clocks": clocks,
            "paper_context": PAPER_CONTEXT,
        }
        print(json.dumps(out), flush=True)
    if dist.is_initialized():
        dist.destroy_process_group()
    return 0


if __name__ == "__main__":
    sys.exit(main())
