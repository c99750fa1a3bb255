"""bench.py -- headline benchmark of the B200 hot path (one JSON line on rank 0).

Workload = BASELINE.json configs[1] (the config the metric is quoted on):
C2 128^3 voxels, occupancy Bernoulli(0.7) in {1, 1e-3} from seed 0, nu = 0.3.
  (a) headline: one "step" = one assembly-free K.u with u ~ N(0,1) (seed 1);
      metric = hex matvec GDOF/s = N_dofs / device time per step.
  (b) secondary: one deflated PCG solve, x=0 clamped, f ~ N(0,1) (seed 2) on
      the free DOFs, 4^3 agglomerates, tol 1e-8 -- plus the same solve on C1
      and the C4 geometry (the north star's target workload).
Timing: W >= 3 warm-up steps; each timed step is bracketed by CUDA events on
the launching stream and preceded by an untimed 512 MB L2 flush (the C2
working set, ~120 MB, fits in the 126 MB L2). Multi-GPU: the path shards by
independent solves (load cases / adjoints), so N ranks run N replicas with no
data-path collective; time = max over ranks, value = sum of the replicas.

--impl reference: the reference's CPU algorithm for the same metric (the
oracle's C port of numba apply_block24, all host cores), rank 0 only.
"""

from __future__ import annotations

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

N_C2 = 128
METRIC = "hex matvec GDOF/s"
# the workload both arms report (identical dict, so the driver sees the same config)
CONFIG = {"workload": "C2(a) 128^3 Bernoulli(0.7) K.u (BASELINE configs[1])", "n": N_C2,
          "n_dofs": 3 * (N_C2 + 1) ** 3, "n_elems": N_C2 ** 3, "parallelism": "replicas (one per GPU)"}
# fp64 operations per element the mode-space matvec executes (csrc/matvec.cu:
# xy forward 24, z butterfly 24, occupancy scaling 8, mode operator 33, z
# inverse + carry 36, xy inverse 24, four-way node sum 9): its own issue bound
MATVEC_FP64_OPS = 158


def parse(argv=None):
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=200)
    ap.add_argument("--warmup", type=int, default=10)
    ap.add_argument("--impl", default="b200", choices=["b200", "reference"])
    ap.add_argument("--no-secondary", action="store_true")
    ap.add_argument("--no-cpu-baseline", action="store_true")
    return ap.parse_args(argv)


def dist_env():
    return (int(os.environ.get("RANK", "0")), int(os.environ.get("WORLD_SIZE", "1")),
            int(os.environ.get("LOCAL_RANK", "0")))


def replica_workload(rank: int, world: int) -> dict:
    """Every rank runs the full single-GPU workload (replicas only: the path has
    no exchange step). Returned for logging / tests."""
    return {"rank": rank, "world": world, "n": N_C2, "seeds": (0, 1)}


def max_over_ranks(value: float, device=None) -> float:
    """Max of a float over the process group (NCCL on GPU, gloo on CPU)."""
    import torch
    import torch.distributed as dist

    if not (dist.is_available() and dist.is_initialized()) or dist.get_world_size() == 1:
        return float(value)
    t = torch.tensor([float(value)], dtype=torch.float64, device=device or "cpu")
    dist.all_reduce(t, op=dist.ReduceOp.MAX)
    return float(t.item())


def c2_inputs(n=N_C2):
    occ = np.where(np.random.default_rng(0).random(n ** 3) < 0.7, 1.0, 1e-3)
    u = np.random.default_rng(1).standard_normal(3 * (n + 1) ** 3)
    return occ, u


def load_peaks():
    try:
        with open(os.path.join(ROOT, "MEASURED_PEAKS.json")) as fh:
            return float(json.load(fh)["hbm_gbs"]), "measured (MEASURED_PEAKS.json)"
    except Exception:
        return 6650.0, "fallback (B200_PROFILING.md)"


def ncu_traffic(*names: str):
    """DRAM bytes per launch of the matvec from the committed ncu summary
    (the first of `names` present: the latest capture first)."""
    try:
        with open(os.path.join(ROOT, "profiles", "ncu_summary.json")) as fh:
            d = json.load(fh)
        for name in names:
            if name in d:
                return d[name].get("dram_bytes_per_launch")
    except Exception:
        pass
    return None


class ClockSampler:
    """nvidia-smi clocks / throttle reasons sampled during the timed region."""

    FIELDS = ("clocks.sm,clocks.max.sm,clocks_event_reasons.hw_slowdown,clocks_event_reasons.hw_thermal_slowdown,"
              "clocks_event_reasons.sw_thermal_slowdown,clocks_event_reasons.sw_power_cap")
    NAMES = ("hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap")

    def __init__(self, index=0):
        self.index, self.samples, self._stop, self._t = index, [], threading.Event(), None

    def _run(self):
        while not self._stop.is_set():
            try:
                out = subprocess.run(["nvidia-smi", "-i", str(self.index), f"--query-gpu={self.FIELDS}",
                                      "--format=csv,noheader,nounits"], capture_output=True, text=True, timeout=5)
                vals = [v.strip() for v in out.stdout.strip().split(",")]
                if len(vals) == 6:
                    self.samples.append(vals)
            except Exception:
                pass
            self._stop.wait(0.05)

    def __enter__(self):
        self._t = threading.Thread(target=self._run, daemon=True)
        self._t.start()
        return self

    def __exit__(self, *a):
        self._stop.set()
        if self._t:
            self._t.join(timeout=10)

    def summary(self):
        if not self.samples:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["nvidia-smi unavailable"], "samples": 0}

        def num(x):
            try:
                return float(x)
            except ValueError:
                return None

        sm = [v for v in (num(s[0]) for s in self.samples) if v is not None]
        mx = [v for v in (num(s[1]) for s in self.samples) if v is not None]
        reasons = sorted({self.NAMES[i] for s in self.samples for i in range(4) if s[2 + i].lower() == "active"})
        return {"sm_mhz": float(np.median(sm)) if sm else None, "sm_max_mhz": max(mx) if mx else None,
                "reasons": reasons, "samples": len(self.samples)}


def cpu_baseline_matvec(occ, u, n=N_C2, budget_s=12.0):
    """The reference's CPU kernel (C port of apply_block24, all host threads),
    bounded sample of the same workload."""
    from oracle import topovox_oracle as O

    O.build_lib()
    cores = O.lib().oracle_max_threads()
    op = O.Operator(n, n, n, 1.0, occ)
    op.apply(u)
    times, t0 = [], time.perf_counter()
    while time.perf_counter() - t0 < budget_s and len(times) < 200:
        t = time.perf_counter()
        op.apply(u)
        times.append(time.perf_counter() - t)
    return {"value": u.size / float(np.median(times)) / 1e9, "unit": "GDOF/s", "cores": cores, "kind": "port",
            "sample": f"{len(times)} x K.u at 128^3 (C port of numba apply_block24, {cores} threads, median)"}


def run_reference(args):
    rank, world, _ = dist_env()
    if rank != 0:
        return
    occ, u = c2_inputs()
    base = cpu_baseline_matvec(occ, u, budget_s=max(5.0, min(60.0, 0.3 * (args.steps + args.warmup))))
    line = {
        "impl": "reference", "metric": METRIC, "value": base["value"], "unit": "GDOF/s", "n_gpus": args.gpus,
        "steps": args.steps, "warmup": args.warmup, "higher_is_better": True, "scaling": "weak",
        "vs_baseline": None, "dtype": "f64", "data": "synthetic",
        "config": dict(CONFIG),
        "cpu_baseline": base,
        "e2e": {"value": base["value"], "unit": "GDOF/s", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
    }
    print(json.dumps(line), flush=True)


def pcie_bound(torch, nd, stream, e2e_val, reps=20):
    """The e2e step's own bound: its H2D + D2H bytes at the concurrent
    (both-direction) pinned copy rate measured here with plain copies."""
    h = torch.empty(nd, dtype=torch.float64).pin_memory()
    h2 = torch.empty(nd, dtype=torch.float64).pin_memory()
    d1 = torch.empty(nd, dtype=torch.float64, device="cuda")
    d2 = torch.empty(nd, dtype=torch.float64, device="cuda")
    s1, s2 = torch.cuda.Stream(), torch.cuda.Stream()
    for _ in range(2):
        torch.cuda.synchronize()
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        a.record(stream)
        for _ in range(reps):
            with torch.cuda.stream(s1):
                d1.copy_(h, non_blocking=True)
            with torch.cuda.stream(s2):
                h2.copy_(d2, non_blocking=True)
        for st in (s1, s2):
            stream.wait_stream(st)
        b.record(stream)
        torch.cuda.synchronize()
    gbs = 2 * 8 * nd * reps / (a.elapsed_time(b) / 1e3) / 1e9
    bound = gbs * 1e9 / (2 * 8 * nd) * nd / 1e9  # GDOF/s if every step moved only its bytes at that rate
    return {"copy_gbs_both_ways": gbs, "bound_gdofs": bound, "frac": e2e_val / bound}


def device_timed(stream, fn, steps, flush):
    import torch

    starts = [torch.cuda.Event(enable_timing=True) for _ in range(steps)]
    ends = [torch.cuda.Event(enable_timing=True) for _ in range(steps)]
    for i in range(steps):
        flush.fill_(float(i))
        starts[i].record(stream)
        fn()
        ends[i].record(stream)
    torch.cuda.synchronize()
    return np.array([s.elapsed_time(e) for s, e in zip(starts, ends)])


def main():
    args = parse()
    if args.impl == "reference":
        run_reference(args)
        return
    import torch

    rank, world, local = dist_env()
    if world > 1:
        import torch.distributed as dist

        torch.cuda.set_device(local)
        dist.init_process_group("nccl")
    else:
        torch.cuda.set_device(0)
    import paper_2203_15115_b200 as tv
    from paper_2203_15115_b200 import _lib, fea

    occ, u = c2_inputs()
    d = tv.Domain(N_C2, N_C2, N_C2, 1.0)
    op = fea.StiffnessOperator(d, tv.Topology(d, occ), tv.Material(E=1.0, nu=0.3), ())
    ud = torch.from_numpy(u).cuda()
    yd = torch.empty_like(ud)
    flush = torch.empty(512 * 1024 * 1024 // 4, dtype=torch.float32, device="cuda")
    stream = torch.cuda.current_stream()
    p64 = float(_lib.lib().tvb_fp64_peak_tflops(stream.cuda_stream))

    def step():
        op.apply_device(ud, yd)

    # clock ramp (not a step): ~0.3 s of device writes so the SM clock is at
    # its loaded value before the warm-up steps (a short run otherwise times
    # its first steps at ramping clocks)
    t_ramp = time.perf_counter()
    while time.perf_counter() - t_ramp < 0.3:
        for _ in range(8):
            flush.fill_(1.0)
        torch.cuda.synchronize()
    for i in range(max(3, args.warmup)):
        flush.fill_(float(i))
        step()
    torch.cuda.synchronize()
    if world > 1:
        torch.distributed.barrier()
    with ClockSampler(local) as clk:
        times_ms = device_timed(stream, step, args.steps, flush)
    if world > 1:
        torch.distributed.barrier()
    t_total = max_over_ranks(float(times_ms.sum()) / 1e3, device="cuda")
    step_stats = {"mean_ms": float(times_ms.mean()), "median_ms": float(np.median(times_ms)),
                  "p10_ms": float(np.percentile(times_ms, 10)), "p90_ms": float(np.percentile(times_ms, 90)),
                  "min_ms": float(times_ms.min()), "max_ms": float(times_ms.max())}
    nd, ne = d.n_dofs, d.n_elems
    value = world * nd * args.steps / t_total / 1e9
    ms_per_step = t_total * 1e3 / args.steps

    # end to end through the public API with pinned HOST buffers: every step
    # copies its input vector host->device and its K.u device->host inside the
    # timed region. StiffnessOperator.apply_host_batch streams the steps'
    # vectors through the double-buffered slab pipeline (vector v's H2D
    # overlaps vector v-1's D2H); apply_host (one synchronous call per step)
    # is reported beside it.
    u_pin = torch.from_numpy(u).pin_memory()
    y_pin = torch.empty(nd, dtype=torch.float64).pin_memory()
    e2e_steps = max(5, min(args.steps, 50))
    op.apply_host_batch([u_pin] * 3, [y_pin] * 3)  # warm (workspace, streams)
    op.apply_host(u_pin, y_pin)
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record(stream)
    op.apply_host_batch([u_pin] * e2e_steps, [y_pin] * e2e_steps)
    e1.record(stream)
    torch.cuda.synchronize()
    e2e_s = max_over_ranks(e0.elapsed_time(e1) / 1e3, device="cuda")
    e2e_val = world * nd * e2e_steps / e2e_s / 1e9
    e0.record(stream)
    for _ in range(e2e_steps):
        op.apply_host(u_pin, y_pin)  # one synchronous call per step
    e1.record(stream)
    torch.cuda.synchronize()
    e2e_single = world * nd * e2e_steps / max_over_ranks(e0.elapsed_time(e1) / 1e3, device="cuda") / 1e9

    hbm, peak_kind = load_peaks()
    alg_bytes = 8.0 * (2 * nd + ne)
    achieved = alg_bytes / (ms_per_step / 1e3) / 1e9
    flops_dense = 1152.0 * ne
    t_star = max(flops_dense / (p64 * 1e12), alg_bytes / (hbm * 1e9)) if p64 > 0 else None
    # the executed kernel's own bound: its bytes at HBM bandwidth vs its fp64
    # instructions at the fp64 pipe rate (P64 counts an FMA as 2 flops, and a
    # DADD / DMUL issues at the DFMA rate, so the op rate is P64 / 2)
    t_hbm = alg_bytes / (hbm * 1e9)
    t_fp64 = MATVEC_FP64_OPS * ne / (p64 / 2.0 * 1e12) if p64 > 0 else 0.0
    t_own = max(t_hbm, t_fp64)
    line = {
        "metric": METRIC, "value": value, "unit": "GDOF/s", "n_gpus": world, "steps": args.steps,
        "warmup": args.warmup, "ms_per_step": ms_per_step, "higher_is_better": True, "scaling": "weak",
        "vs_baseline": None, "dtype": "f64", "data": "synthetic (seeded Bernoulli(0.7) occupancy, N(0,1) u)",
        "config": dict(CONFIG),
        "l2": "flushed (512 MB write) before every timed step",
        "step_stats": step_stats,
        "value_median": nd / (step_stats["median_ms"] / 1e3) / 1e9 * world,
        "roofline": {
            "bound": "hbm", "achieved": achieved, "peak": hbm, "unit": "GB/s", "frac": achieved / hbm,
            "traffic": ncu_traffic("k_matvec_c2_r02d", "k_matvec_c2_r02c", "k_matvec_c2_r02b", "k_matvec_c2_r02", "k_matvec_c2_r01c", "k_matvec_c2_r01b", "k_matvec_c2"),
            "peak_kind": peak_kind, "alg_bytes_per_launch": alg_bytes,
            "own_bound": {"t_hbm_us": t_hbm * 1e6, "t_fp64_issue_us": t_fp64 * 1e6,
                          "fp64_ops_per_elem": MATVEC_FP64_OPS, "p64_tflops_live": p64,
                          "frac": t_own / (ms_per_step / 1e3),
                          "frac_median": t_own / (step_stats["median_ms"] / 1e3)},
            "north_star": {"definition": "max(1152*Ne FMA-flops / P64, bytes / HBM) (dense-k0 flops the "
                                         "mode-space kernel does not execute)",
                           "t_star_us": t_star * 1e6 if t_star else None,
                           "frac": (t_star / (ms_per_step / 1e3)) if t_star else None},
        },
        "e2e": {"value": e2e_val, "unit": "GDOF/s", "h2d_bytes_per_step": 8 * nd, "d2h_bytes_per_step": 8 * nd,
                "api": "StiffnessOperator.apply_host_batch (pinned host vectors, %d steps)" % e2e_steps,
                "single_call_value": e2e_single, "pcie": pcie_bound(torch, nd, stream, e2e_val)},
        "gpu_launches": args.steps,  # one k_matvec launch per timed step
        "clocks": clk.summary(),
    }
    if rank == 0 and not args.no_secondary:
        line["secondary"] = secondary_solves(tv, fea, torch, p64, hbm)
        line["secondary"]["C4_two_load_cases_batched"] = secondary_batch(tv, fea, torch, p64, hbm)
        line["secondary"]["C4_optimizer"] = secondary_optimizer(torch)
        line["secondary"]["C4_fields"] = secondary_fields(tv, fea, torch, hbm)
        if world == 1 and not args.no_cpu_baseline:
            line["secondary"]["C1_optimizer"] = secondary_optimizer_c1(torch)
    if rank == 0 and world == 1 and not args.no_cpu_baseline:
        try:
            line["cpu_baseline"] = cpu_baseline_matvec(occ, u)
        except Exception as exc:  # pragma: no cover
            line["cpu_baseline"] = {"error": repr(exc)}
    if rank == 0:
        print(json.dumps(line), flush=True)
    if world > 1:
        torch.distributed.destroy_process_group()


def _case(tv, d, lo=None, hi=None):
    nx, ny, nz = d.nx, d.ny, d.nz
    loads = ((tv.RegionSelector("box", min=lo, max=hi), (0, 0, -1), "total"),) if lo is not None else ()
    return tv.LoadCase("c", dirichlet=((tv.RegionSelector("box", min=(0, 0, 0), max=(0, ny, nz)), (1, 1, 1)),),
                       loads=loads)


def dpcg_roofline(d, defl, us_per_iter, p64, hbm):
    """Roofline of one deflated-PCG iteration: the sum of each
    stage's algorithmic minimum time --
      2 matvecs (q = A p, t = A z)   each max(1152 Ne flops / P64, 8 (6 Nn + Ne) B / HBM)
      fused update x, r, z + dots    8 vectors x 8*3Nn B / HBM
      restriction W^T (t + beta q)   2 vectors / HBM
      coarse solve                   factor bytes (G, [Z|-G^T], top inverse) / HBM
      prolongation p = z + beta p - W nu   3 vectors / HBM
    -- against the measured time per iteration."""
    vec = 8.0 * d.n_dofs
    t_mv = max(1152.0 * d.n_elems / (p64 * 1e12), 8.0 * (2 * d.n_dofs + d.n_elems) / (hbm * 1e9))
    coarse_bytes = float(defl.nd.bytes) if defl.nd is not None else 8.0 * defl.n_vectors ** 2
    stages = {"matvec_x2": 2 * t_mv, "update": 8 * vec / (hbm * 1e9), "restrict": 2 * vec / (hbm * 1e9),
              "coarse": coarse_bytes / (hbm * 1e9), "prolong": 3 * vec / (hbm * 1e9)}
    t_star = sum(stages.values())
    # SURVEY §8(d) definition (reference algorithm): K p + (KW)^T z as W^T(K z)
    # (bytes 8(N_d + N_e)), 11 vector passes (88 B/DOF), banded coarse sweeps
    # 16 n_c w with w = 6 (m1 m2 + m1 + 1), m sorted ascending.
    m = sorted(defl.grid)
    w = 6 * (m[0] * m[1] + m[0] + 1)
    t_r = max(1152.0 * d.n_elems / (p64 * 1e12), 8.0 * (d.n_dofs + d.n_elems) / (hbm * 1e9))
    t_survey = t_mv + t_r + 88.0 * d.n_dofs / (hbm * 1e9) + 16.0 * 6 * defl.n_blocks * w / (hbm * 1e9)
    # Executed-algorithm bound: the matvec at the bound of the kernel
    # that actually runs -- max(its bytes / HBM, its ~158 fp64 operations per
    # element at the fp64 pipe's lane rate) -- instead of the dense-k0 flops;
    # the other stages as above.
    t_mv_own = max(8.0 * (2 * d.n_dofs + d.n_elems) / (hbm * 1e9),
                   MATVEC_FP64_OPS * d.n_elems / (0.5 * p64 * 1e12))
    t_exec = t_star - 2 * t_mv + 2 * t_mv_own
    return {"t_star_us": t_star * 1e6, "frac": t_star * 1e6 / us_per_iter,
            "stages_us": {k: round(v * 1e6, 2) for k, v in stages.items()},
            "survey_def": {"t_star_us": t_survey * 1e6, "frac": t_survey * 1e6 / us_per_iter},
            "executed_def": {"t_star_us": t_exec * 1e6, "frac": t_exec * 1e6 / us_per_iter,
                             "matvec_own_bound_us": round(t_mv_own * 1e6, 2)},
            "p64_tflops": p64, "hbm_gbs": hbm}


def secondary_solves(tv, fea, torch, p64, hbm):
    """Deflated PCG solves (device-timed): C1, C3, the C4 geometry (north-star
    target), C5 (load case 1: 5x5 patch) and C2(b) (BASELINE configs[1] part
    b; C2(b) and C5 are infeasible for the reference's dense coarse factor)."""
    out = {}
    specs = [("C1_40x20x20_b4", (40, 20, 20), 4, (40, 10, 10), (40, 10, 10), None),
             ("C3_80x40x40_b4", (80, 40, 40), 4, (80, 20, 20), (80, 20, 20), None),
             ("C4a_160x80x80_b8", (160, 80, 80), 8, (160, 39, 39), (160, 41, 41), None),
             ("C5_320x160x160_b8", (320, 160, 160), 8, (320, 78, 78), (320, 82, 82), None),
             ("C2b_128^3_b4_bernoulli", (128, 128, 128), 4, None, None, "c2b")]
    for name, dims, b, lo, hi, kind in specs:
        try:
            d = tv.Domain(*dims, 1.0)
            case = _case(tv, d, lo, hi)
            fixed = tv.dirichlet_dofs(d, case)
            if kind == "c2b":
                occ = np.where(np.random.default_rng(0).random(d.n_elems) < 0.7, 1.0, 1e-3)
                f = np.random.default_rng(2).standard_normal(d.n_dofs)
                f[fixed] = 0.0
            else:
                occ = np.ones(d.n_elems)
                f = tv.assemble_force(d, case)
            fd = torch.from_numpy(f).cuda()
            op = fea.StiffnessOperator(d, tv.Topology(d, occ), tv.Material(E=1.0, nu=0.3), fixed)
            torch.cuda.synchronize()
            t0 = time.perf_counter()
            defl = fea.build_deflation(d, op.topology, fixed, b)
            defl.prepare(op)
            torch.cuda.synchronize()
            setup = time.perf_counter() - t0
            if kind != "c2b":
                fea.solve_static(op, fd, tol=1e-8, deflation=defl)  # warm (graph capture)
            a, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            a.record()
            r = fea.solve_static(op, fd, tol=1e-8, deflation=defl)
            e.record()
            torch.cuda.synchronize()
            ms = a.elapsed_time(e)
            us_it = 1e3 * ms / max(r.iterations, 1)
            out[name] = {"iterations": r.iterations, "solve_ms": ms, "us_per_iter": us_it,
                         "setup_s": setup, "residual": r.residual, "J": float(fd @ r.u),
                         "n_coarse": defl.n_vectors,
                         "coarse": "nested dissection" if defl.nd is not None else "dense inverse",
                         "roofline": dpcg_roofline(d, defl, us_it, p64, hbm)}
            if name.startswith("C1"):
                # plain Jacobi PCG on the device, and the reference's CPU path
                # (oracle port) for both solves, timed here on this box's cores
                a.record()
                rp = fea.solve_static(op, fd, tol=1e-8)
                e.record()
                torch.cuda.synchronize()
                out[name]["plain"] = {"iterations": rp.iterations, "solve_ms": a.elapsed_time(e)}
                out[name]["cpu"] = cpu_c1_solves(d, occ, fixed, f, setup + ms / 1e3, ms, a.elapsed_time(e))
            del op, defl, r
            torch.cuda.empty_cache()
        except Exception as exc:
            out[name] = {"error": repr(exc)[:300]}
    return out


def cpu_c1_solves(d, occ, fixed, f, gpu_total_s, gpu_dpcg_ms, gpu_plain_ms):
    """The reference's CPU path for the C1 solves (oracle port: numba kernels
    restated in C with all host threads, scipy dense Cholesky coarse solve,
    the reference's loop), timed in the same run on this box's host cores."""
    try:
        from oracle import topovox_oracle as O

        O.build_lib()
        ref = O.Operator(d.nx, d.ny, d.nz, d.h, occ, dirichlet=fixed)
        t0 = time.perf_counter()
        defl = O.Deflation(ref, 4)
        defl.prepare()
        t1 = time.perf_counter()
        _, it, _ = O.solve_static(ref, f, tol=1e-8, deflation=defl)
        t2 = time.perf_counter()
        _, itp, _ = O.solve_static(ref, f, tol=1e-8)
        t3 = time.perf_counter()
        cores = O.lib().oracle_max_threads()
        return {"kind": "port", "cores": cores,
                "sample": f"C1 DPCG (b = 4, build + prepare + solve) and plain Jacobi PCG, tol 1e-8, {cores} threads",
                "dpcg_setup_s": t1 - t0, "dpcg_solve_s": t2 - t1, "dpcg_iterations": it,
                "plain_solve_s": t3 - t2, "plain_iterations": itp,
                "speedup_dpcg_solve": (t2 - t1) / (gpu_dpcg_ms / 1e3),
                "speedup_dpcg_with_setup": (t2 - t0) / gpu_total_s,
                "speedup_plain": (t3 - t2) / (gpu_plain_ms / 1e3)}
    except Exception as exc:  # pragma: no cover
        return {"error": repr(exc)[:300]}


def secondary_optimizer_c1(torch, outer=3):
    """BASELINE configs[0] (C1) optimizer, first `outer` outer iterations, on
    the device and on the reference's CPU path (the oracle's SPEC-restated
    loop over the oracle FEA, all host threads) in the same run."""
    try:
        from oracle import topovox_oracle as O
        from paper_2203_15115_b200 import optimize as opt
        from paper_2203_15115_b200.mesh import assemble_force, dirichlet_dofs

        prob = opt.cantilever_problem(40, 20, 20, (40, 10, 10), (40, 10, 10),
                                      constraints=[opt.ConstraintSpec("compliance", 1.6)])
        cfg = opt.OptimizerConfig(ersatz=1e-3, block=4, max_outer=outer)
        opt.run(prob, opt.OptimizerConfig(ersatz=1e-3, block=4, max_outer=1))  # warm (graphs, plans)
        torch.cuda.synchronize()
        t0 = time.perf_counter()
        _, hist, _ = opt.run(prob, cfg)
        torch.cuda.synchronize()
        t_gpu = time.perf_counter() - t0
        case = prob.load_cases[0]
        fixed, f = dirichlet_dofs(prob.domain, case), assemble_force(prob.domain, case)
        t0 = time.perf_counter()
        _, hist_r, _ = O.run_optimizer(40, 20, 20, [(fixed, f)], [{"kind": "compliance", "alpha": 1.6, "case": 0}],
                                       block=4, ersatz=1e-3, max_outer=outer)
        t_cpu = time.perf_counter() - t0
        return {"outer_iterations": len(hist), "gpu_s": t_gpu, "solves": sum(h.solves for h in hist),
                "volumes": [round(h.v, 6) for h in hist], "volumes_oracle": [round(h["v"], 6) for h in hist_r],
                "cpu": {"kind": "port", "cores": O.lib().oracle_max_threads(), "seconds": t_cpu,
                        "sample": f"first {outer} outer iterations of the C1 run (base analysis included)"},
                "speedup": t_cpu / t_gpu}
    except Exception as exc:  # pragma: no cover
        return {"error": repr(exc)[:300]}


def secondary_fields(tv, fea, torch, hbm):
    """Per-element sensitivity / level-set kernels at the C4 geometry
    (160x80x80, full solid), device-timed (CUDA events, mean of 20 launches
    after warm-up), each against its algorithmic HBM bytes (DESIGN.md §3,
    SURVEY §8(d)): element state + T_J + p-norm sums 8 (N_d + 3 N_e); adjoint
    right-hand side 8 (2 N_d + N_e); T_sigma 8 (2 N_d + 2 N_e); combine of two
    fields (max-abs passes + weighted sum) 8 * 5 N_e; threshold select 16 N_e
    (read the level set, write the occupancy)."""
    try:
        from paper_2203_15115_b200 import levelset, sensitivity

        d = tv.Domain(160, 80, 80, 1.0)
        case = _case(tv, d, (160, 39, 39), (160, 41, 41))
        fixed = tv.dirichlet_dofs(d, case)
        op = fea.StiffnessOperator(d, tv.Topology(d, np.ones(d.n_elems)), tv.Material(E=1.0, nu=0.3), fixed)
        u = torch.from_numpy(np.random.default_rng(3).standard_normal(d.n_dofs)).cuda()
        lam = torch.from_numpy(np.random.default_rng(4).standard_normal(d.n_dofs)).cuda()
        nd, ne = d.n_dofs, d.n_elems
        _, tj, sums = sensitivity.element_fields_device(op, u, 8)
        ts = sensitivity.stress_sensitivity(op, u, lam)
        design = torch.from_numpy(d.design_mask.astype(np.uint8)).cuda()
        ls = levelset.combine_device([tj, ts], [2.0, 1.0])
        stages = {
            "element_state_TJ_pnorm": (lambda: sensitivity.element_fields_device(op, u, 8), 8.0 * (nd + 3 * ne)),
            "adjoint_rhs": (lambda: sensitivity.adjoint_rhs_device(op, u, 8, sums), 8.0 * (2 * nd + ne)),
            "stress_sensitivity": (lambda: sensitivity.stress_sensitivity(op, u, lam), 8.0 * (2 * nd + 2 * ne)),
            "combine_2_fields": (lambda: levelset.combine_device([tj, ts], [2.0, 1.0]), 8.0 * 5 * ne),
            "threshold_select": (lambda: levelset.extract_device(d, ls, 0.5, 1e-3, design), 16.0 * ne),
        }
        out = {}
        a, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        for name, (fn, nbytes) in stages.items():
            for _ in range(3):
                fn()
            torch.cuda.synchronize()
            a.record()
            for _ in range(20):
                fn()
            e.record()
            torch.cuda.synchronize()
            us = 1e3 * a.elapsed_time(e) / 20
            out[name] = {"us": us, "alg_bytes": nbytes, "gbs": nbytes / (us / 1e6) / 1e9,
                         "frac_hbm": nbytes / (us / 1e6) / 1e9 / hbm}
        out["note"] = ("timed through the public device API (includes its small allocations / host "
                       "round trips: the select reads its 4-word state back)")
        return out
    except Exception as exc:  # pragma: no cover
        return {"error": repr(exc)[:300]}


def secondary_optimizer(torch, outer=3):
    """The north-star loop itself: augmented-Lagrangian level-set optimizer on
    BASELINE configs[3] (160x80x80, two load cases, compliance <= 2 J0 and
    p-norm (p = 8) stress <= 1.2x per case, 8^3 agglomerates). Host-driven
    loop over device analyses; wall time per outer iteration after the first
    (which includes the full-domain baseline analyses), device synchronised."""
    try:
        from paper_2203_15115_b200 import optimize as opt

        prob = opt.cantilever_problem(160, 80, 80, (160, 39, 39), (160, 41, 41), force=(0, 0, -1),
                                      extra_cases=[("case2", (160, 39, 39), (160, 41, 41), (0, -1, 0))],
                                      constraints=[opt.ConstraintSpec("compliance", 2.0, load_case="load"),
                                                   opt.ConstraintSpec("compliance", 2.0, load_case="case2"),
                                                   opt.ConstraintSpec("pnorm_stress", 1.2, load_case="load", p=8),
                                                   opt.ConstraintSpec("pnorm_stress", 1.2, load_case="case2", p=8)])
        stamps = []

        def cb(rec):
            torch.cuda.synchronize()
            stamps.append((time.perf_counter(), rec.solves, rec.inner_iters, rec.accepted))

        torch.cuda.synchronize()
        t0 = time.perf_counter()
        opt.run(prob, opt.OptimizerConfig(ersatz=1e-3, block=8, max_outer=outer), callback=cb)
        per = [b[0] - a[0] for a, b in zip(stamps, stamps[1:])]
        return {"outer_iterations": len(stamps), "first_s": stamps[0][0] - t0 if stamps else None,
                "s_per_outer_after_first": float(np.mean(per)) if per else None,
                "solves_per_outer": [st[1] for st in stamps], "inner_per_outer": [st[2] for st in stamps],
                "note": "solves of one topology run as multi-RHS batches (load cases, then adjoints)"}
    except Exception as exc:
        return {"error": repr(exc)[:300]}


def secondary_batch(tv, fea, torch, p64, hbm):
    """Multi-RHS batching: the two load cases of BASELINE
    configs[3] ((0,0,-1) and (0,-1,0) over the 3x3 patch of the x=160 face) on
    the full-solid C4 geometry, solved one after the other (solve_static) and
    as one batch (solve_static_batch); device-timed, tol 1e-8."""
    try:
        d = tv.Domain(160, 80, 80, 1.0)
        fs = []
        for fv in ((0, 0, -1), (0, -1, 0)):
            case = tv.LoadCase("c", dirichlet=((tv.RegionSelector("box", min=(0, 0, 0), max=(0, 80, 80)), (1, 1, 1)),),
                               loads=((tv.RegionSelector("box", min=(160, 39, 39), max=(160, 41, 41)), fv, "total"),))
            fs.append(torch.from_numpy(tv.assemble_force(d, case)).cuda())
        fixed = tv.dirichlet_dofs(d, case)
        op = fea.StiffnessOperator(d, tv.Topology(d, np.ones(d.n_elems)), tv.Material(E=1.0, nu=0.3), fixed)
        defl = fea.build_deflation(d, op.topology, fixed, 8)
        defl.prepare(op)
        fea.solve_static_batch(op, fs, tol=1e-8, deflation=defl)  # warm
        for f in fs:
            fea.solve_static(op, f, tol=1e-8, deflation=defl)

        def timed(fn):
            a, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            torch.cuda.synchronize()
            a.record()
            out = fn()
            e.record()
            torch.cuda.synchronize()
            return a.elapsed_time(e), out

        t_seq, rs = timed(lambda: [fea.solve_static(op, f, tol=1e-8, deflation=defl) for f in fs])
        t_bat, rb = timed(lambda: fea.solve_static_batch(op, fs, tol=1e-8, deflation=defl))
        its = [r.iterations for r in rb]
        us_rhs = 1e3 * t_bat / sum(its)
        # per-RHS roofline of the batch: every stage per RHS except the coarse
        # solve, whose factor is read once per iteration for all RHS
        rf = dpcg_roofline(d, defl, us_rhs, p64, hbm)
        st = rf["stages_us"]
        t_rhs = st["matvec_x2"] + st["update"] + st["restrict"] + st["prolong"] + st["coarse"] / len(fs)
        return {"iterations": its, "sequential_ms": t_seq, "batch_ms": t_bat, "speedup": t_seq / t_bat,
                "us_per_rhs_iter": us_rhs,
                "roofline": {"t_star_us_per_rhs": t_rhs, "frac": t_rhs / us_rhs,
                             "note": "DPCG iteration roofline (DESIGN.md §7) with the coarse factor shared by the RHS"},
                "bitwise_equal_to_single": all(torch.equal(x.u, y.u) for x, y in zip(rs, rb))}
    except Exception as exc:
        return {"error": repr(exc)[:300]}


if __name__ == "__main__":
    main()
