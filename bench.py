"""bench.py -- headline benchmark of the B200 hot path (one JSON line on rank 0).

Workload (BASELINE.json configs[1], the config the metric is quoted on):
C2(a) 128^3 voxels, occupancy Bernoulli(0.7) in {1, 1e-3} from seed 0, nu=0.3,
u ~ N(0,1) from seed 1. One "step" = one assembly-free K.u (the hex matvec).
metric: hex matvec GDOF/s (N_d per step / device time). Secondary keys report
the deflated-PCG solve (BASELINE configs C1 / C4) measured the same way.

Timing: W warm-up steps, then K timed steps; each step is bracketed by CUDA
events on the launching stream and preceded by an (untimed) 512 MB L2 flush,
since the C2 working set (~120 MB) fits in the 126 MB L2. Multi-GPU: every
rank runs an independent replica (the path shards by independent solves;
there is no collective on the data path), time = max over ranks.

--impl reference: the reference's CPU algorithm (the oracle's C port of
apply_block24, all host cores) on the same workload.
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


def parse():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=200)
    ap.add_argument("--warmup", type=int, default=10)
    ap.add_argument("--impl", default="b200", choices=["b200", "reference"])
    ap.add_argument("--no-secondary", action="store_true")
    ap.add_argument("--no-cpu-baseline", action="store_true")
    return ap.parse_args()


def dist_env():
    rank = int(os.environ.get("RANK", "0"))
    world = int(os.environ.get("WORLD_SIZE", "1"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    return rank, world, local


def c2_inputs(n=N_C2):
    ne = n ** 3
    occ = np.where(np.random.default_rng(0).random(ne) < 0.7, 1.0, 1e-3)
    nd = 3 * (n + 1) ** 3
    u = np.random.default_rng(1).standard_normal(nd)
    return occ, u


def load_peaks():
    try:
        with open(os.path.join(ROOT, "MEASURED_PEAKS.json")) as fh:
            p = json.load(fh)
        return float(p["hbm_gbs"]), "measured"
    except Exception:
        return 6650.0, "fallback"


class ClockSampler:
    """nvidia-smi clocks / throttle reasons sampled during the timed region."""

    FIELDS = ("clocks.sm,clocks.max.sm,clocks_event_reasons.hw_slowdown,clocks_event_reasons.hw_thermal_slowdown,"
              "clocks_event_reasons.sw_thermal_slowdown,clocks_event_reasons.sw_power_cap")

    def __init__(self, index=0):
        self.index = index
        self.samples = []
        self._stop = threading.Event()
        self._t = None

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
            self._stop.wait(0.1)

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
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["nvidia-smi unavailable"]}
        sm = [float(s[0]) for s in self.samples if s[0].replace(".", "").isdigit()]
        mx = [float(s[1]) for s in self.samples if s[1].replace(".", "").isdigit()]
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        reasons = sorted({names[i] for s in self.samples for i in range(4) if s[2 + i].lower() == "active"})
        return {"sm_mhz": float(np.median(sm)) if sm else None, "sm_max_mhz": max(mx) if mx else None,
                "reasons": reasons, "samples": len(self.samples)}


def cpu_baseline_matvec(occ, u, n=N_C2, budget_s=12.0):
    """The reference's CPU kernel (C port of apply_block24, all host threads)
    on the same workload, bounded sample."""
    from oracle import topovox_oracle as O

    O.build_lib()
    cores = O.lib().oracle_max_threads()
    op = O.Operator(n, n, n, 1.0, occ)
    op.apply(u)  # warm
    t0 = time.perf_counter()
    reps = 0
    times = []
    while time.perf_counter() - t0 < budget_s and reps < 200:
        t = time.perf_counter()
        op.apply(u)
        times.append(time.perf_counter() - t)
        reps += 1
    nd = u.size
    best = min(times)
    return {"value": nd / float(np.median(times)) / 1e9, "best": nd / best / 1e9, "unit": "GDOF/s", "cores": cores,
            "kind": "port", "sample": f"{reps} x K.u at 128^3 (C port of numba apply_block24, median)"}


def run_reference(args):
    rank, world, _ = dist_env()
    if rank != 0:
        return
    occ, u = c2_inputs()
    base = cpu_baseline_matvec(occ, u, budget_s=max(5.0, min(60.0, 0.5 * (args.steps + args.warmup))))
    line = {
        "impl": "reference", "metric": "hex matvec GDOF/s", "value": base["value"], "unit": "GDOF/s",
        "n_gpus": args.gpus, "steps": args.steps, "warmup": args.warmup, "higher_is_better": True,
        "scaling": "weak", "vs_baseline": None, "dtype": "f64", "data": "synthetic",
        "config": {"workload": "C2(a) 128^3 Bernoulli(0.7) K.u", "n": N_C2},
        "cpu_baseline": {k: base[k] for k in ("value", "unit", "cores", "kind", "sample")},
        "e2e": {"value": base["value"], "unit": "GDOF/s", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
    }
    print(json.dumps(line), flush=True)


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
    from paper_2203_15115_b200 import fea

    occ, u = c2_inputs()
    d = tv.Domain(N_C2, N_C2, N_C2, 1.0)
    op = fea.StiffnessOperator(d, tv.Topology(d, occ), tv.Material(E=1.0, nu=0.3), ())
    ud = torch.from_numpy(u).cuda()
    yd = torch.empty_like(ud)
    flush = torch.empty(512 * 1024 * 1024 // 4, dtype=torch.float32, device="cuda")
    stream = torch.cuda.current_stream()

    def step():
        op.apply_device(ud, yd)

    for _ in range(max(3, args.warmup)):
        flush.fill_(1.0)
        step()
    torch.cuda.synchronize()
    if world > 1:
        torch.distributed.barrier()
    starts = [torch.cuda.Event(enable_timing=True) for _ in range(args.steps)]
    ends = [torch.cuda.Event(enable_timing=True) for _ in range(args.steps)]
    with ClockSampler(local) as clk:
        torch.cuda.synchronize()
        for i in range(args.steps):
            flush.fill_(float(i))
            starts[i].record(stream)
            step()
            ends[i].record(stream)
        torch.cuda.synchronize()
    if world > 1:
        torch.distributed.barrier()
    times_ms = np.array([s.elapsed_time(e) for s, e in zip(starts, ends)])
    t_total = float(times_ms.sum()) / 1e3
    if world > 1:
        tt = torch.tensor([t_total], device="cuda", dtype=torch.float64)
        torch.distributed.all_reduce(tt, op=torch.distributed.ReduceOp.MAX)
        t_total = float(tt.item())
    nd, ne = d.n_dofs, d.n_elems
    value = world * nd * args.steps / t_total / 1e9
    ms_per_step = t_total * 1e3 / args.steps

    # end-to-end through the public API with host buffers (pinned)
    u_pin = torch.from_numpy(u).pin_memory()
    y_pin = torch.empty(nd, dtype=torch.float64).pin_memory()
    e2e_steps = max(5, min(args.steps, 50))
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record(stream)
    for _ in range(e2e_steps):
        udev = u_pin.to("cuda", non_blocking=True)
        out = op.apply_device(udev)
        y_pin.copy_(out, non_blocking=True)
    e1.record(stream)
    torch.cuda.synchronize()
    e2e_s = e0.elapsed_time(e1) / 1e3
    e2e_val = world * nd * e2e_steps / e2e_s / 1e9

    hbm, peak_kind = load_peaks()
    alg_bytes = 8.0 * (2 * nd + ne)
    achieved = alg_bytes / (ms_per_step / 1e3) / 1e9
    line = {
        "metric": "hex matvec GDOF/s", "value": value, "unit": "GDOF/s", "n_gpus": world, "steps": args.steps,
        "warmup": args.warmup, "ms_per_step": ms_per_step, "higher_is_better": True, "scaling": "weak",
        "vs_baseline": None, "dtype": "f64", "data": "synthetic (seeded Bernoulli(0.7) occupancy, N(0,1) u)",
        "config": {"workload": "C2(a) 128^3 Bernoulli(0.7) K.u", "n": N_C2, "n_dofs": nd, "n_elems": ne,
                   "l2": "flushed (512 MB write) before every timed step", "parallelism": f"replicas x{world}"},
        "roofline": {"bound": "hbm", "achieved": achieved, "peak": hbm, "unit": "GB/s", "frac": achieved / hbm,
                     "traffic": None, "peak_kind": peak_kind,
                     "alg_bytes_per_launch": alg_bytes,
                     "dense_k0_equiv_tflops": 1152.0 * ne / (ms_per_step / 1e3) / 1e12},
        "e2e": {"value": e2e_val, "unit": "GDOF/s", "h2d_bytes_per_step": 8 * nd, "d2h_bytes_per_step": 8 * nd},
        "gpu_launches": args.steps,
        "clocks": clk.summary(),
    }
    if rank == 0 and not args.no_secondary:
        line["secondary"] = secondary_solves(tv, fea, torch)
    if rank == 0 and world == 1 and not args.no_cpu_baseline:
        try:
            line["cpu_baseline"] = {k: v for k, v in cpu_baseline_matvec(occ, u).items() if k != "best"}
        except Exception as exc:  # pragma: no cover
            line["cpu_baseline"] = {"error": repr(exc)}
    if rank == 0:
        print(json.dumps(line), flush=True)
    if world > 1:
        torch.distributed.destroy_process_group()


def secondary_solves(tv, fea, torch):
    """DPCG solve times on the C1 and C4-geometry cantilevers (device-timed)."""
    out = {}
    for name, (nx, ny, nz), b, lo, hi in [
        ("C1_40x20x20_b4", (40, 20, 20), 4, (40, 10, 10), (40, 10, 10)),
        ("C4a_160x80x80_b8", (160, 80, 80), 8, (160, 39, 39), (160, 41, 41)),
    ]:
        try:
            d = tv.Domain(nx, ny, nz, 1.0)
            case = tv.LoadCase("c", dirichlet=((tv.RegionSelector("box", min=(0, 0, 0), max=(0, ny, nz)), (1, 1, 1)),),
                               loads=((tv.RegionSelector("box", min=lo, max=hi), (0, 0, -1), "total"),))
            fixed = tv.dirichlet_dofs(d, case)
            f = torch.from_numpy(tv.assemble_force(d, case)).cuda()
            op = fea.StiffnessOperator(d, tv.Topology(d, np.ones(d.n_elems)), tv.Material(E=1.0, nu=0.3), fixed)
            t0 = time.perf_counter()
            defl = fea.build_deflation(d, op.topology, fixed, b)
            defl.prepare(op)
            torch.cuda.synchronize()
            setup = time.perf_counter() - t0
            fea.solve_static(op, f, tol=1e-8, deflation=defl)  # warm (graph capture etc.)
            torch.cuda.synchronize()
            t0 = time.perf_counter()
            r = fea.solve_static(op, f, tol=1e-8, deflation=defl)
            torch.cuda.synchronize()
            solve = time.perf_counter() - t0
            out[name] = {"iterations": r.iterations, "solve_s": solve, "us_per_iter": 1e6 * solve / max(r.iterations, 1),
                         "setup_s": setup, "J": float(f @ r.u), "n_coarse": defl.n_vectors}
        except Exception as exc:
            out[name] = {"error": repr(exc)[:300]}
    return out


if __name__ == "__main__":
    main()
