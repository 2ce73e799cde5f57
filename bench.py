#!/usr/bin/env python
"""bench.py — HVP GDOF/s + sparse-tangent assembly ms on B200 (BASELINE.json metric).

Workload (default): BASELINE cfg 3 — 3D compressible neo-Hookean block [0,1]^3, 150^3
Kuhn-Tet4 cells (10,328,853 DOFs, 20.25M elements), perturbed interior nodes (a = 0.1,
seed 13), roller stretch eps = 0.05 (DESIGN.md §8 input recipe).  One step = one pass of
the whole per-iteration hot path over that mesh, all through the C ABI:
    fem_energy -> fem_residual (BC) -> fem_hvp (BC) -> fem_assemble_csr (BC, Alg. 2)
    -> fem_spmv
Pattern + coloring (setup) and the solves (a12/a13) are timed
separately in the same run.  `value` = HVP GDOF/s = DOFs x HVP calls / HVP device time
(CUDA events on the launching stream), whole job over all ranks.

--impl reference times the CPU oracle (the reference arm of this tier) on a bounded
sample of the same workload.
"""
from __future__ import annotations

import argparse
import json
import os
import subprocess
import sys
import time

import numpy as np

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

import fem_inputs as fi  # noqa: E402

METRIC = "HVP GDOF/s + sparse-tangent assembly ms vs DOFs, 1/2/4/8 B200, % HBM peak"
UNIT = "GDOF/s"


def parse():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=20)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--config", type=int, default=3, choices=[2, 3, 5, 6],
                    help="BASELINE cfg 2 / 3 / 5; 6 = unstructured 3D NH Delaunay block (not a "
                         "BASELINE config: the general-mesh paths at scale; --n = interior points "
                         "in thousands, default 1000)")
    ap.add_argument("--n", type=int, default=None, help="override the mesh size (cells per side)")
    ap.add_argument("--assemble-mode", default="auto", choices=["auto", "batched", "literal", "rows", "scatter", "colored"])
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--no-solve", action="store_true")
    ap.add_argument("--setup-reps", type=int, default=5, help="timed pattern + coloring runs")
    ap.add_argument("--profile-step", action="store_true", help="one step only (for ncu)")
    ap.add_argument("--scaling", default="weak", choices=["weak", "strong"],
                    help="weak: one cfg-3-sized z-slab per GPU (N = 1: cfg 3 itself); strong: "
                         "BASELINE cfg 4 (255x255x256 cells, 50.5M DOFs) cut into N z-slabs")
    return ap.parse_args()


def delaunay_workload(n_pts):
    """cfg 6 (reading R11): qhull Delaunay of seeded points + a surface grid, NH,
    roller stretch; state noise 1e-4 h (Delaunay slivers invert under a 1e-2 h jitter)."""
    side = max(4, int(round(n_pts ** (1.0 / 3.0) / 2.5)))
    mesh = fi.roller_bc(fi.delaunay_tet4(n_pts, side, 7).copy_with(material=fi.NEO_HOOKEAN), 0.05)
    h = mesh.length / n_pts ** (1.0 / 3.0)
    z = fi.lift(mesh, fi.generic_state(mesh, 5, eps=0.05, noise=1e-4, h=h))
    v = fi.random_direction(mesh.n_total, 4)
    name = (f"unstructured 3D NH Delaunay block: {n_pts} interior points + {side}^3 surface grid, "
            f"{mesh.n_total} DOFs, {mesh.n_elems} tets (not a BASELINE config)")
    return mesh, name, z, v


def workload(cfg, n):
    if cfg == 6:
        return delaunay_workload(1000 * (n or 1000))
    mesh = fi.config_mesh(cfg, n=n)
    name = {2: "cfg2: 2D NH plate Tri3", 3: "cfg3: 3D NH block Kuhn-Tet4",
            5: "cfg5: 2D LE + periodic MPC Tri3"}[cfg]
    h = mesh.length / max(mesh.shape)
    z = fi.lift(mesh, fi.generic_state(mesh, 5, eps=0.05, noise=0.01, h=h))
    v = fi.random_direction(mesh.n_total, 4)
    return mesh, name, z, v


# ------------------------------------------------------------------ clocks
class Clocks:
    FIELDS = ("clocks.sm,clocks.max.sm,power.draw,clocks_event_reasons.active,"
              "clocks_event_reasons.hw_slowdown,clocks_event_reasons.hw_thermal_slowdown,"
              "clocks_event_reasons.sw_thermal_slowdown,clocks_event_reasons.sw_power_cap")

    def __init__(self, index):
        self.index = index
        self.proc = None

    def start(self):
        try:
            self.proc = subprocess.Popen(
                ["nvidia-smi", "-i", str(self.index), f"--query-gpu={self.FIELDS}",
                 "--format=csv,noheader,nounits", "-lms", "50"],
                stdout=subprocess.PIPE, stderr=subprocess.DEVNULL, text=True)
        except OSError:
            self.proc = None

    def stop(self):
        if self.proc is None:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["nvidia-smi unavailable"]}
        self.proc.terminate()
        out, _ = self.proc.communicate(timeout=10)
        rows = [[c.strip() for c in l.split(",")] for l in out.strip().splitlines() if l.strip()]
        rows = [r for r in rows if len(r) >= 8]
        if not rows:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["no samples"]}
        sm = [float(r[0]) for r in rows if r[0].replace(".", "").isdigit()]
        mx = [float(r[1]) for r in rows if r[1].replace(".", "").isdigit()]
        names = ("hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap")
        reasons = sorted({names[i] for r in rows for i in range(4) if r[4 + i] == "Active"})
        load = [s for s in sm if s > 0.5 * max(sm)] if sm else []
        return {"sm_mhz": float(np.median(load)) if load else None,
                "sm_max_mhz": max(mx) if mx else None, "reasons": reasons,
                "samples": len(rows)}


# ------------------------------------------------------------------ oracle (CPU) arm
def host_cpu():
    model = "unknown"
    try:
        for line in open("/proc/cpuinfo"):
            if line.startswith("model name"):
                model = line.split(":", 1)[1].strip()
                break
    except OSError:
        pass
    return {"model": model, "host_cores": os.cpu_count()}


def _time_best(fn, budget):
    """best of >= 1 runs, repeated while the budget (s) lasts (at most 3 runs)."""
    best, spent, runs = float("inf"), 0.0, 0
    while runs < 3 and (runs == 0 or spent + best <= budget):
        t0 = time.perf_counter()
        fn()
        dt = time.perf_counter() - t0
        best, spent, runs = min(best, dt), spent + dt, runs + 1
    return best


def oracle_sample(cfg, budget=4.0):
    """The oracle as it stands (plain C, one thread, pinned to one core) on a bounded
    sub-block of the workload: energy, residual, HVP, pattern and coloring,
    each the best of up to 3 runs within `budget` seconds; throughput = DOFs / op time
    (reading C18).  Returns the cpu_baseline object (value = HVP GDOF/s)."""
    import oracle
    try:
        os.sched_setaffinity(0, {sorted(os.sched_getaffinity(0))[0]})
    except (AttributeError, OSError):
        pass
    if cfg == 6:
        mesh, _, z, v = delaunay_workload(30000)
    else:
        n = {3: 40, 2: 400, 5: 400}[cfg]
        mesh = fi.config_mesh(cfg, n=n)
        h = mesh.length / max(mesh.shape)
        z = fi.lift(mesh, fi.generic_state(mesh, 5, eps=0.05, noise=0.01, h=h))
        v = fi.random_direction(mesh.n_total, 4)
    o = oracle.Oracle(mesh)
    N = mesh.n_total
    t0 = time.perf_counter()
    ops = {"energy": lambda: o.energy(z), "residual": lambda: o.residual(z, bc=True),
           "hvp": lambda: o.hvp(z, v, bc=True)}
    secs = {k: _time_best(f, budget) for k, f in ops.items()}
    o.hvp(z, v, bc=True)

    def pattern():
        o._pattern = None
        o.sparsity()

    secs["pattern"] = _time_best(pattern, budget)
    rp, ci = o.sparsity()
    secs["coloring"] = _time_best(lambda: oracle.color(rp, ci), budget)
    total = time.perf_counter() - t0
    per_op = {k: {"s": t, "GDOF/s": N / t / 1e9} for k, t in secs.items()}
    return {"value": N / secs["hvp"] / 1e9, "unit": UNIT, "cores": 1, "kind": "oracle",
            "sample": f"oracle (plain C, 1 thread pinned to one core) on the "
                      f"{'30k-point Delaunay' if cfg == 6 else f'{n}^{mesh.dim}-cell'} "
                      f"sub-block of the workload ({N} DOFs, nnz {len(ci)}): energy, residual, "
                      f"HVP (value), pattern, coloring, best of <= 3 runs each; {total:.1f} s",
            "n_dofs": N, "per_op": per_op, "host_cpu": host_cpu(), "oracle_threads": 1}


def run_reference(args):
    rank = int(os.environ.get("RANK", "0"))
    if rank != 0:
        return
    import oracle
    os.sched_setaffinity(0, {sorted(os.sched_getaffinity(0))[0]})
    n = {3: 40, 2: 400, 5: 400}[args.config]
    mesh = fi.config_mesh(args.config, n=n)
    h = mesh.length / max(mesh.shape)
    z = fi.lift(mesh, fi.generic_state(mesh, 5, eps=0.05, noise=0.01, h=h))
    v = fi.random_direction(mesh.n_total, 4)
    o = oracle.Oracle(mesh)
    for _ in range(args.warmup):
        o.hvp(z, v, bc=True)
    t0 = time.perf_counter()
    for _ in range(args.steps):
        o.hvp(z, v, bc=True)
    dt = time.perf_counter() - t0
    val = mesh.n_total * args.steps / dt / 1e9
    sample = (f"fem_ref_hvp on the {n}^{mesh.dim}-cell sub-block of the workload "
              f"({mesh.n_total} DOFs) per step")
    print(json.dumps({
        "impl": "reference", "metric": METRIC, "value": val, "unit": UNIT, "n_gpus": args.gpus,
        "steps": args.steps, "warmup": args.warmup, "ms_per_step": 1e3 * dt / args.steps,
        "higher_is_better": True, "scaling": "weak", "vs_baseline": None, "dtype": "f64",
        "data": "synthetic",
        "config": {"workload": workload_name(args.config), "n_dofs_sample": mesh.n_total},
        "cpu_baseline": {"value": val, "unit": UNIT, "cores": 1, "kind": "oracle", "sample": sample,
                         "host_cpu": host_cpu()},
        "e2e": {"value": val, "unit": UNIT, "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0}}))


def scaling_plan(mode: str, world: int, n=None) -> dict:
    """Global problem and per-rank z-slab of the multi-GPU bench.

    weak:   every rank owns an n x n x n Kuhn block (n = 150: cfg 3 per GPU) stacked in z;
            the global block is n x n x (n P) cells.
    strong: BASELINE cfg 4, 255 x 255 x 256 cells (50,528,256 DOFs) whatever P is; rank r
            owns cells z in [r 256/P, (r+1) 256/P).
    DOFs = 3 (nx+1)(ny+1)(nz+1); elements = 6 nx ny nz."""
    if mode == "strong":
        nx = ny = 255 if n is None else n
        nz_total = 256 if n is None else n + 1
        if nz_total % world:
            raise SystemExit(f"strong scaling: {nz_total} z-cells do not split into {world} slabs")
        nzr = nz_total // world
        name = (f"strong scaling: BASELINE cfg4 3D NH block {nx}x{ny}x{nz_total} Kuhn-Tet4 cells "
                f"split into {world} z-slabs of {nzr} cells, perturbed a=0.1, roller eps=0.05, "
                f"NCCL halo add")
        seed = 14
    else:
        nx = ny = nzr = 150 if n is None else n
        nz_total = nzr * world
        name = (f"weak scaling: {world} z-slabs of {nx}^3 Kuhn-Tet4 cells (cfg 3 per GPU), "
                f"3D NH, perturbed a=0.1, roller eps=0.05, NCCL halo add")
        seed = 13
    nodes = (nx + 1) * (ny + 1) * (nz_total + 1)
    return {"mode": mode, "nx": nx, "ny": ny, "nz_total": nz_total, "nz_per_rank": nzr,
            "n_global_nodes": nodes, "n_global_dofs": 3 * nodes,
            "n_global_elems": 6 * nx * ny * nz_total, "workload": name, "seed": seed}


def workload_name(cfg):
    return {3: "BASELINE cfg3: 3D compressible neo-Hookean block, 150^3 Kuhn-Tet4 cells, "
               "10,328,853 DOFs, perturbed a=0.1, roller eps=0.05",
            2: "BASELINE cfg2: 2D compressible neo-Hookean plate, 706^2 Tri3 cells, 999,698 DOFs",
            5: "BASELINE cfg5: 2D linear elastic + periodic MPC",
            6: "unstructured 3D NH Delaunay block (not a BASELINE config)"}[cfg]


# ------------------------------------------------------------------ B200 arm
# Algorithmic bytes per DOF (compulsory traffic, geometry recomputed from
# coordinates; 3D Kuhn: 2 tets/DOF, 1/3 node/DOF) and FP64 flops per element.
# FP64 flops per element of the minimal formulations (FMA = 2; SURVEY §8(d2) counting
# scalar, geometry recomputed): energy / residual / HVP; assembly = per-element tangent
# context (~ residual + spatial gradients) + the (d+1)^2 blocks K_ab (d^2 entries, 6 flops
# each, plus the G_a.G_b dot) — DESIGN.md §5.
# B200 nominal FP64: 148 SMs x 64 DFMA/clk x 2 flops x 1.965 GHz (B200_PROFILING.md unit counts)
FP64_NOMINAL = 148 * 64 * 2 * 1.965e9 / 1e12
FLOPS = {(3, 1): (189, 266, 457), (3, 0): (156, 204, 258), (2, 1): (59, 79, 141), (2, 0): (54, 64, 80)}


def algorithmic(mesh, nnz, C, mode):
    N, E, d = mesh.n_total, mesh.n_elems, mesh.dim
    nen = d + 1
    conn = 4 * nen * E
    coords = 8 * d * mesh.n_nodes
    vec = 8 * N
    fe, fr, fh = FLOPS[(d, mesh.material)]
    f_ctx = fr + 2 * d * d * nen
    f_blocks = nen * nen * (2 * d + 6 * d * d)
    asm_bytes = conn + coords + vec + 8 * nnz                          # inputs + vals written once
    if mode in ("batched", "literal") or (mode == "auto" and d == 2 and mesh.n_mpc):  # J_comp
        asm_bytes += 2 * 8 * N * C + nnz * (4 + 4)
    return {
        "energy": {"bytes": conn + coords + vec, "flops": fe * E},
        "residual": {"bytes": conn + coords + vec + 2 * vec, "flops": fr * E},  # r zero + write
        "hvp": {"bytes": conn + coords + 2 * vec + 2 * vec, "flops": fh * E},   # u, v; y zero + write
        "assemble": {"bytes": asm_bytes, "flops": (f_ctx + f_blocks) * E},
        # node-block SpMV (no multipliers): vals + one neighbour id per D x D block; plain
        # CSR otherwise (vals + col_idx + row_ptr)
        "spmv": {"bytes": (nnz * 8 + 4 * nnz // (d * d) + 8 * (mesh.n_nodes + 1) if not mesh.n_mpc
                           else nnz * 12 + 8 * (N + 1)) + 2 * vec, "flops": 2 * nnz},
    }


def main():
    args = parse()
    if args.impl == "reference":
        return run_reference(args)
    import torch
    import torch.distributed as dist
    from paper_2602_12365_b200 import build as fbuild
    from paper_2602_12365_b200 import fem

    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    if world != args.gpus:
        raise SystemExit(f"WORLD_SIZE={world} but --gpus {args.gpus}: launch N > 1 under "
                         f"torch.distributed.run with --nproc-per-node N")
    torch.cuda.set_device(local)
    if world > 1:
        dist.init_process_group("nccl", device_id=torch.device("cuda", local))
    fbuild.build()

    comm = None
    plan = scaling_plan(args.scaling, world, args.n)
    if args.scaling == "strong" or world > 1:
        # element partition into z-slabs: weak = one cfg-3-sized slab per rank,
        # strong = BASELINE cfg 4 (255 x 255 x 256 cells) cut into slabs of 256/P cells.
        # One halo add per residual / HVP / SpMV over NCCL; states drawn per global node so
        # shared DOFs agree on every rank and every P computes the same global problem.
        from paper_2602_12365_b200 import dist as fd
        if args.config != 3:
            raise SystemExit("multi-GPU bench runs the 3D Kuhn slabs (cfg 3 weak / cfg 4 strong)")
        mesh, gids = fd.slab_mesh(plan["nx"], plan["ny"], plan["nz_per_rank"], world, rank,
                                  perturb_a=0.1, seed=plan["seed"])
        hplan = None
        if world > 1:
            all_ids = [None] * world
            dist.all_gather_object(all_ids, gids)
            hplan = fd.halo_plan(all_ids, rank)
            del all_ids
            uid = [fem.nccl_unique_id() if rank == 0 else None]
            dist.broadcast_object_list(uid, src=0)
            comm = fem.nccl_comm_init(uid[0], rank, world)
            plan["nccl_comm_count"] = fem.nccl_comm_count(comm)
            assert plan["nccl_comm_count"] == world
        h = 1.0 / max(plan["nx"], plan["ny"], plan["nz_total"])
        gz = np.random.default_rng(5).uniform(-0.01 * h, 0.01 * h, size=(plan["n_global_nodes"], 3))
        gv = np.random.default_rng(4).uniform(-1, 1, size=(plan["n_global_nodes"], 3))
        z = fi.lift(mesh, (fi.affine_field(mesh, np.diag([0.05, 0.0, 0.0])).reshape(-1, 3)
                           + gz[gids]).ravel())
        v = gv[gids].ravel()
        del gz, gv
        wname = plan["workload"]
        prob = fem.Problem(mesh, plan=hplan, nccl_comm=comm)
    else:
        mesh, wname, z, v = workload(args.config, args.n)
        prob = fem.Problem(mesh)
    N = mesh.n_total
    zt = torch.as_tensor(z, device="cuda")
    vt = torch.as_tensor(v, device="cuda")
    stream = torch.cuda.current_stream()

    # ---- setup: pattern + coloring (a7, a8), timed separately.  A tiny problem of the same
    # element / material runs first so lazy CUDA module loading is not charged to setup.
    tiny = fi.grid_tet4(3, 3, 3) if mesh.dim == 3 else fi.grid_tri3(4, 4)
    tiny = fi.roller_bc(tiny.copy_with(material=mesh.material), 0.01)
    tp = fem.Problem(tiny)
    tz = torch.zeros(tiny.n_total, dtype=torch.float64, device="cuda")
    tp.nnz()
    tp.color()
    tp.energy(tz), tp.residual(tz, bc=True), tp.hvp(tz, tz, bc=True)
    tp.spmv(tp.assemble_csr(tz, bc=True, mode=args.assemble_mode), tz)
    del tp
    ev = lambda: torch.cuda.Event(enable_timing=True)  # noqa: E731
    torch.cuda.synchronize()
    e0, e1, e2 = ev(), ev(), ev()
    e0.record()
    nnz = prob.nnz()
    e1.record()
    colors, C = prob.color()
    e2.record()
    torch.cuda.synchronize()
    setup = {"pattern_ms_first": e0.elapsed_time(e1), "coloring_ms_first": e1.elapsed_time(e2),
             "nnz": nnz, "n_colors": C}
    if world == 1:
        # 3 warm-up runs, then the median of >= 5; each run is a fresh problem
        # on the same mesh (the pattern and colors are per problem), timed with CUDA events
        samples = {"pattern_ms": [], "coloring_ms": []}
        for rep in range(3 + args.setup_reps):
            p2 = fem.Problem(mesh)
            torch.cuda.synchronize()
            e0.record()
            p2.nnz()
            e1.record()
            p2.color()
            e2.record()
            torch.cuda.synchronize()
            if rep >= 3:
                samples["pattern_ms"].append(e0.elapsed_time(e1))
                samples["coloring_ms"].append(e1.elapsed_time(e2))
            del p2
        for key, xs in samples.items():
            setup[key] = float(np.median(xs))
            setup[key + "_samples"] = xs
        setup["note"] = ("*_first: the bench problem's own first call (first touch of the "
                         "multi-GB allocations); median of fresh problems after 3 warm-ups")

    energy = torch.empty(1, dtype=torch.float64, device="cuda")
    r = torch.empty(N, dtype=torch.float64, device="cuda")
    y = torch.empty(N, dtype=torch.float64, device="cuda")
    ys = torch.empty(N, dtype=torch.float64, device="cuda")
    vals = torch.empty(nnz, dtype=torch.float64, device="cuda")
    phases = ("energy", "residual", "hvp", "assemble", "spmv")
    mode = args.assemble_mode

    def step(evs=None):
        def mark(i):
            if evs is not None:
                evs[i].record(stream)
        mark(0)
        prob.energy(zt, out=energy)
        mark(1)
        prob.residual(zt, bc=True, out=r)
        mark(2)
        prob.hvp(zt, vt, bc=True, out=y)
        mark(3)
        prob.assemble_csr(zt, bc=True, mode=mode, out=vals)
        mark(4)
        prob.spmv(vals, vt, out=ys)
        mark(5)

    if args.profile_step:
        # one warm step (lazy setup), then exactly one step inside the profiler range
        # (ncu --profile-from-start off captures only that)
        step()
        torch.cuda.synchronize()
        torch.cuda.profiler.start()
        step()
        torch.cuda.synchronize()
        torch.cuda.profiler.stop()
        prob.check()
        return

    for _ in range(args.warmup):
        step()
    torch.cuda.synchronize()
    prob.check()

    clocks = Clocks(local)
    clocks.start()
    time.sleep(0.2)
    events = [[ev() for _ in range(6)] for _ in range(args.steps)]
    if world > 1:
        dist.barrier()
    torch.cuda.synchronize()
    t_start, t_end = ev(), ev()
    t_start.record(stream)
    for it in range(args.steps):
        step(events[it])
    t_end.record(stream)
    torch.cuda.synchronize()
    if world > 1:
        dist.barrier()
    time.sleep(0.1)
    clk = clocks.stop()
    prob.check()
    total_ms = t_start.elapsed_time(t_end)
    per = {ph: sum(events[it][i].elapsed_time(events[it][i + 1]) for it in range(args.steps))
           for i, ph in enumerate(phases)}
    if world > 1:
        t = torch.tensor([total_ms] + [per[p] for p in phases], dtype=torch.float64, device="cuda")
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        total_ms = float(t[0])
        per = {p: float(t[i + 1]) for i, p in enumerate(phases)}
    K = args.steps
    n_global = plan["n_global_dofs"] if (world > 1 or args.scaling == "strong") else N
    hvp_ms = per["hvp"] / K
    value = n_global / (hvp_ms * 1e-3) / 1e9

    # ---- A/B variants of the hot kernels (outside the timed region, same inputs)
    def time_call(fn, reps=5):
        fn()
        torch.cuda.synchronize()
        a, b = ev(), ev()
        a.record(stream)
        for _ in range(reps):
            fn()
        b.record(stream)
        torch.cuda.synchronize()
        return a.elapsed_time(b) / reps

    prob.linearize(zt)
    e1 = torch.empty(1, dtype=torch.float64, device=zt.device)
    ab = {
        "hvp_tiles_ms": time_call(lambda: prob.hvp(zt, vt, bc=True, out=y)),
        # the per-element reference metric mu vol G_a.G_b, 1/det J read from a cache computed
        # once per problem (Alg. 1's precomputed geometry) instead of recomputed per call
        "hvp_reference_metric_ms": time_call(
            lambda: prob.hvp(zt, vt, bc=True, out=y, flags=fem.REFERENCE_METRIC)),
        "residual_reference_metric_ms": time_call(
            lambda: prob.residual(zt, bc=True, out=r, flags=fem.REFERENCE_METRIC)),
        "hvp_linearized_ms": time_call(lambda: prob.hvp(zt, vt, bc=True, out=y, flags=fem.LINEARIZED)),
        "linearize_ms": time_call(lambda: prob.linearize(zt)),
        "hvp_baseline_scatter_ms": time_call(
            lambda: prob.hvp(zt, vt, bc=True, out=y, flags=fem.BASELINE_SCATTER)),
        "hvp_deterministic_ms": time_call(
            lambda: prob.hvp(zt, vt, bc=True, out=y, flags=fem.DETERMINISTIC)),
        "energy_plus_residual_ms": time_call(
            lambda: (prob.energy(zt, out=e1), prob.residual(zt, bc=True, out=r))),
        "energy_residual_one_pass_ms": time_call(
            lambda: prob.energy_residual(zt, bc=True, out_energy=e1, out=r)),
        "residual_baseline_scatter_ms": time_call(
            lambda: prob.residual(zt, bc=True, out=r, flags=fem.BASELINE_SCATTER)),
        # geometry streamed per element (Alg. 1's gather, 80 B / tet,
        # one TMA bulk copy per tile) instead of recomputed from the coordinates
        "hvp_stream_geom_ms": time_call(lambda: prob.hvp(zt, vt, bc=True, out=y, flags=fem.STREAM_GEOM)),
        "residual_stream_geom_ms": time_call(
            lambda: prob.residual(zt, bc=True, out=r, flags=fem.STREAM_GEOM)),
        # A/B 1(C): element-colored conflict-free passes (plain stores, no atomics)
        "hvp_colored_scatter_ms": time_call(
            lambda: prob.hvp(zt, vt, bc=True, out=y, flags=fem.COLORED_SCATTER)),
        "residual_colored_scatter_ms": time_call(
            lambda: prob.residual(zt, bc=True, out=r, flags=fem.COLORED_SCATTER)),
        # the same at tile granularity: tile-colored passes, plain boundary writes
        "hvp_tile_colored_ms": time_call(
            lambda: prob.hvp(zt, vt, bc=True, out=y, flags=fem.TILE_COLORED)),
        "residual_tile_colored_ms": time_call(
            lambda: prob.residual(zt, bc=True, out=r, flags=fem.TILE_COLORED)),
        "assemble_batched_ms": time_call(lambda: prob.assemble_csr(zt, bc=True, mode="batched", out=vals), 2),
        "assemble_rows_ms": time_call(lambda: prob.assemble_csr(zt, bc=True, mode="rows", out=vals), 2),
        "assemble_literal_ms": time_call(lambda: prob.assemble_csr(zt, bc=True, mode="literal", out=vals), 1),
        "assemble_scatter_add_ms": time_call(lambda: prob.assemble_csr(zt, bc=True, mode="scatter", out=vals), 2),
        "assemble_colored_fused_ms": time_call(lambda: prob.assemble_csr(zt, bc=True, mode="colored", out=vals), 2),
    }
    prob.check()

    # ---- gpu launches in one step (torch profiler, outside the timed region)
    launches_per_step = None
    kernel_names = {}
    try:
        from torch.profiler import ProfilerActivity, profile
        with profile(activities=[ProfilerActivity.CUDA]) as prof:
            step()
            torch.cuda.synchronize()
        for e in prof.events():
            if e.device_type.name == "CUDA" and not e.name.startswith(("Memset", "Memcpy")):
                kernel_names[e.name] = kernel_names.get(e.name, 0) + 1
        launches_per_step = sum(kernel_names.values())
    except Exception as ex:  # profiler unavailable: count stays None
        kernel_names = {"error": str(ex)}

    # ---- e2e: the HVP through the C ABI with host buffers, copies inside the timed region.
    # Every step copies its z, v from pinned host memory and reads its y back; steps are
    # pipelined over two buffer sets and three streams (H2D copy engine, compute, D2H copy
    # engine), so step k+1's upload and step k-1's download overlap step k's HVP.
    zh = torch.from_numpy(z).pin_memory()
    vh = torch.from_numpy(v).pin_memory()
    yh = [torch.empty(N, dtype=torch.float64).pin_memory() for _ in range(2)]
    zd = [torch.empty_like(zt) for _ in range(2)]
    vd = [torch.empty_like(vt) for _ in range(2)]
    yd = [torch.empty_like(y) for _ in range(2)]
    s_up, s_down = torch.cuda.Stream(), torch.cuda.Stream()
    up_done = [torch.cuda.Event() for _ in range(2)]
    comp_done = [torch.cuda.Event() for _ in range(2)]
    down_done = [torch.cuda.Event() for _ in range(2)]
    used = [False, False]

    def e2e_step(k):
        bb = k & 1
        with torch.cuda.stream(s_up):
            if used[bb]:
                s_up.wait_event(comp_done[bb])        # inputs of step k-2 consumed
            zd[bb].copy_(zh, non_blocking=True)
            vd[bb].copy_(vh, non_blocking=True)
            up_done[bb].record(s_up)
        stream.wait_event(up_done[bb])
        if used[bb]:
            stream.wait_event(down_done[bb])          # y of step k-2 downloaded
        prob.hvp(zd[bb], vd[bb], bc=True, out=yd[bb])
        comp_done[bb].record(stream)
        with torch.cuda.stream(s_down):
            s_down.wait_event(comp_done[bb])
            yh[bb].copy_(yd[bb], non_blocking=True)
            down_done[bb].record(s_down)
        used[bb] = True

    for k in range(2):
        e2e_step(k)
    torch.cuda.synchronize()
    a, b = ev(), ev()
    a.record(stream)
    for k in range(K):
        e2e_step(k)
    for bb in range(2):
        stream.wait_event(down_done[bb])
    b.record(stream)
    torch.cuda.synchronize()
    e2e_ms = a.elapsed_time(b) / K
    n_local_sum = N
    if world > 1:  # max over ranks of the device time; bytes summed over ranks
        t = torch.tensor([e2e_ms], dtype=torch.float64, device="cuda")
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        e2e_ms = float(t[0])
        t = torch.tensor([N], dtype=torch.int64, device="cuda")
        dist.all_reduce(t)
        n_local_sum = int(t[0])
    e2e = {"value": n_global / (e2e_ms * 1e-3) / 1e9, "unit": UNIT,
           "h2d_bytes_per_step": 2 * 8 * n_local_sum, "d2h_bytes_per_step": 8 * n_local_sum,
           "what": "fem_hvp with pinned-host z, v copied in and y copied out every step; "
                   "steps pipelined over 2 buffer sets (H2D / compute / D2H streams)"}

    # ---- roofline of the dominant phase
    peaks = {}
    try:
        peaks = json.load(open(os.path.join(ROOT, "MEASURED_PEAKS.json")))
    except Exception:
        pass
    hbm = peaks.get("hbm_gbs")
    hbm_src = "measured (MEASURED_PEAKS.json)" if hbm else "fallback (B200_PROFILING.md)"
    hbm = hbm or 6650.0
    fp64 = None
    try:
        import ctypes
        peak_so = fbuild.build_peak()
        lp = ctypes.CDLL(peak_so)
        lp.fem_peak_fp64_tflops.restype = ctypes.c_double
        fp64 = lp.fem_peak_fp64_tflops(torch.cuda.get_device_properties(local).multi_processor_count)
    except Exception:
        pass
    fp64_src = "measured (bench_tools/peak.cu DFMA)" if fp64 else "nominal 148 SM x 64 DFMA x 2 x 1.965 GHz"
    fp64 = fp64 or FP64_NOMINAL
    alg = algorithmic(mesh, nnz, C, mode)
    phase_roofline = {}
    for p in phases:
        ms = per[p] / K
        gbs = alg[p]["bytes"] / (ms * 1e-3) / 1e9
        tfs = alg[p]["flops"] / (ms * 1e-3) / 1e12
        t_hbm = alg[p]["bytes"] / (hbm * 1e9)
        t_alu = alg[p]["flops"] / (fp64 * 1e12)
        phase_roofline[p] = {"ms": ms, "alg_GB": alg[p]["bytes"] / 1e9, "GB/s": gbs,
                             "frac_hbm": gbs / hbm, "alg_GFLOP": alg[p]["flops"] / 1e9,
                             "TFLOP/s": tfs, "frac_fp64": tfs / fp64,
                             "frac_fp64_nominal": tfs / FP64_NOMINAL,
                             "bound": "hbm" if t_hbm >= t_alu else "alu",
                             "frac_of_bound": max(t_hbm, t_alu) / (ms * 1e-3),
                             "share_of_step": per[p] / total_ms}
    # the linearized HVP (Newton-Krylov operator, fem_linearize + FEM_LINEARIZED): compulsory
    # bytes = the cached metric-form tangent (D^2 + 2 + D(D+1)/2 doubles per element) + v read
    # + y zeroed and written; FP64 ~ 130 flops per tet (3D)
    if mesh.material == 1:
        d_ = mesh.dim
        lin_b = 8 * (d_ * d_ + 2 + d_ * (d_ + 1) // 2) * mesh.n_elems + 3 * 8 * N
        ms_l = ab["hvp_linearized_ms"]
        extra_phases = {"hvp_linearized": {
            "ms": ms_l, "alg_GB": lin_b / 1e9, "GB/s": lin_b / (ms_l * 1e-3) / 1e9,
            "frac_hbm": lin_b / (ms_l * 1e-3) / 1e9 / hbm, "gdofs": n_global / (ms_l * 1e-3) / 1e9,
            "what": "FEM_LINEARIZED HVP (cached metric-form tangent, 136 B/tet) - the operator "
                    "of fem_newton_solve's matrix-free CG; A/B timing, 5 calls"}}
    else:
        extra_phases = {}
    dom = max(phases, key=lambda p: per[p])
    pr = phase_roofline[dom]
    if pr["bound"] == "hbm":
        roofline = {"bound": "hbm", "achieved": pr["GB/s"], "peak": hbm, "unit": "GB/s",
                    "frac": pr["frac_hbm"], "peak_source": hbm_src}
    else:
        roofline = {"bound": "alu", "achieved": pr["TFLOP/s"], "peak": fp64, "unit": "TFLOP/s",
                    "frac": pr["frac_fp64"], "peak_source": fp64_src,
                    "peak_nominal": FP64_NOMINAL, "frac_nominal": pr["frac_fp64_nominal"],
                    "frac_hbm": pr["frac_hbm"]}
    traffic = None
    if args.config == 3 and world == 1 and not args.n and args.scaling != "strong":
        try:  # ncu's DRAM bytes of the same launch configuration (profiled on cfg 3 only)
            tj = json.load(open(os.path.join(ROOT, "profiles", "ncu_traffic.json")))
            traffic = tj["dram_bytes_per_launch"].get(dom)
        except Exception:
            pass
    roofline.update({"traffic": traffic, "kernel_phase": dom,
                     "note": "algorithmic bytes/flops per launch / CUDA-event time of the phase; "
                             "traffic from ncu in profiles/"})

    # ---- solves (outside the timed region): CG per-iteration cost and Newton
    solve = {}
    if not args.no_solve:
        b0 = torch.as_tensor(v, device="cuda").clone()
        b0[torch.as_tensor(mesh.dirichlet_dofs.astype(np.int64), device="cuda")] = 0.0
        for op, name in ((0, "cg_hvp"), (1, "cg_csr")):
            # a warm-up solve first (lazy module loading, graph capture), then a timed one;
            # rtol = 0 runs to the cap unless CG reaches its rounding floor (breakdown)
            prob.cg_solve(b0, z=zt, vals=vals, op=op, rtol=0.0, max_iter=64, check_every=32,
                          raise_on_fail=False)
            torch.cuda.synchronize()
            a, b = ev(), ev()
            a.record(stream)
            _, info = prob.cg_solve(b0, z=zt, vals=vals, op=op, rtol=0.0, max_iter=64,
                                    check_every=32, raise_on_fail=False)
            b.record(stream)
            torch.cuda.synchronize()
            solve[name + "_ms_per_iter"] = a.elapsed_time(b) / max(info["iters"], 1)
            solve[name + "_iters_timed"] = info["iters"]
        # affine predictor of the roller stretch (reading R2): eps from the prescribed u_x
        eps = float(mesh.dirichlet_vals.max()) / mesh.length if len(mesh.dirichlet_vals) else 0.0
        z0 = torch.as_tensor(fi.lift(mesh, fi.affine_field(mesh, np.diag([eps] + [0.0] * (mesh.dim - 1)))),
                             device="cuda") if args.config != 5 else None
        if z0 is not None:
            t0 = time.perf_counter()
            zs, info = prob.newton_solve(z0, op=0, cg_rtol=1e-8, rtol=1e-10, atol=1e-14,
                                         check_every=16, raise_on_fail=False)
            torch.cuda.synchronize()
            solve["newton_s"] = time.perf_counter() - t0
            solve["newton"] = {k: info[k] for k in ("iters", "cg_iters", "converged", "res0", "res")}
            # BASELINE cfg 3 as stated: colored sparse tangent + SpMV-CG (Jacobi) per Newton step
            t0 = time.perf_counter()
            zc, infoc = prob.newton_solve(z0, op=1, jacobi=True, cg_rtol=1e-8, rtol=1e-10,
                                          atol=1e-14, check_every=16, raise_on_fail=False)
            torch.cuda.synchronize()
            solve["newton_csr_s"] = time.perf_counter() - t0
            solve["newton_csr"] = {k: infoc[k] for k in ("iters", "cg_iters", "converged", "res0", "res")}
            solve["newton_csr_vs_hvp_maxdiff"] = float((zc - zs).abs().max())
            # inexact Newton-Krylov (Eisenstat-Walker forcing, reading R16): same outer target
            for key, op, jac in (("newton_ew", 0, False), ("newton_csr_ew", 1, True)):
                t0 = time.perf_counter()
                ze, infoe = prob.newton_solve(z0, op=op, jacobi=jac, cg_rtol=1e-8, rtol=1e-10,
                                              atol=1e-14, check_every=16, raise_on_fail=False,
                                              forcing=0.9)
                torch.cuda.synchronize()
                solve[key + "_s"] = time.perf_counter() - t0
                solve[key] = {k: infoe[k] for k in ("iters", "cg_iters", "converged", "res0", "res")}
                solve[key + "_vs_fixed_maxdiff"] = float((ze - zs).abs().max())

    cpu = None
    if not args.no_cpu_baseline and rank == 0 and world == 1:
        cpu = oracle_sample(args.config)

    out = {
        "metric": METRIC, "value": value, "unit": UNIT, "n_gpus": world, "steps": K,
        "warmup": args.warmup, "ms_per_step": total_ms / K, "higher_is_better": True,
        "scaling": args.scaling, "vs_baseline": None, "dtype": "f64", "data": "synthetic",
        "config": {"workload": wname if (args.n or world > 1 or args.scaling == "strong")
                   else workload_name(args.config),
                   "n_dofs": n_global,
                   "n_elems": plan["n_global_elems"] if (world > 1 or args.scaling == "strong")
                   else mesh.n_elems,
                   "nnz": nnz, "n_colors": C,  # rank 0's local CSR when P > 1
                   "assemble_mode": mode, "parallelism": f"element partition x{world} (z-slabs)",
                   "nccl_comm_count": plan.get("nccl_comm_count"),
                   "l2": f"inputs larger than L2 (126 MB): the HVP moves {alg['hvp']['bytes'] / 1e9:.2f} GB per call (algorithmic)"},
        "assembly_ms": per["assemble"] / K,
        "assembly_what": f"mode {mode}: {'row-owner gather of element-Hessian rows (SURVEY §8(f) f1; no J_comp, no colors)' if mode in ('auto', 'rows') else mode}",
        # the paper's colored Alg. 2 (compressed Jacobian by colored HVPs + decompression):
        # the faster of its literal per-color form and the one-sweep form, same run
        "colored_assembly_ms": min(ab["assemble_batched_ms"], ab["assemble_literal_ms"],
                                   ab["assemble_colored_fused_ms"]),
        "residual_gdofs": n_global / (per["residual"] / K * 1e-3) / 1e9,
        "energy_gdofs": n_global / (per["energy"] / K * 1e-3) / 1e9,
        "spmv_ms": per["spmv"] / K,
        "phases": phase_roofline,
        "phases_extra": extra_phases,
        "ab": ab,
        "setup": setup,
        "solve": solve,
        "roofline": roofline,
        "fp64_peak_tflops_measured": fp64,
        "cpu_baseline": cpu,
        "e2e": e2e,
        "gpu_launches": None if launches_per_step is None else launches_per_step * K,
        "kernels_per_step": kernel_names,
        "clocks": clk,
    }
    if rank == 0:
        print(json.dumps(out))
    if comm is not None:
        del prob
        torch.cuda.synchronize()
        fem.nccl_comm_destroy(comm)
    if world > 1:
        dist.destroy_process_group()


if __name__ == "__main__":
    main()
