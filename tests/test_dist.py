"""Multi-process (world_size 2, gloo, CPU) coverage of the N>1 host path of
bench.py: replica assignment and the max-over-ranks timing reduction. The data
path has no collective (replicas only)."""

import os
import socket
import sys

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def _free_port():
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        return s.getsockname()[1]


def _worker(rank, world, port, q):
    sys.path.insert(0, ROOT)
    import torch.distributed as dist

    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port), RANK=str(rank), WORLD_SIZE=str(world))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    import bench

    t = bench.max_over_ranks(1.5 + rank)
    w = bench.replica_workload(rank, world)
    dist.barrier()
    dist.destroy_process_group()
    q.put((rank, t, w))


def test_gloo_two_ranks_max_and_replicas():
    import torch.multiprocessing as mp

    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, 2, port, q)) for r in range(2)]
    for p in procs:
        p.start()
    res = sorted(q.get(timeout=120) for _ in procs)
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    assert [r[1] for r in res] == [2.5, 2.5]
    assert res[0][2]["n"] == res[1][2]["n"] and res[0][2]["seeds"] == res[1][2]["seeds"]


def test_single_process_passthrough():
    sys.path.insert(0, ROOT)
    import bench

    assert bench.max_over_ranks(3.25) == 3.25
    args = bench.parse(["--gpus", "1", "--steps", "5", "--warmup", "3"])
    assert args.steps == 5 and args.warmup == 3 and args.impl == "b200"


@pytest.mark.timeout(300)
def test_reference_arm_cpu(capsys):
    """--impl reference runs the oracle's C port on the host cores and prints
    the contract line (impl, cpu_baseline, e2e) without a GPU."""
    sys.path.insert(0, ROOT)
    import json

    import bench

    import numpy as np

    old = bench.N_C2
    bench.N_C2 = 24  # small grid: the arm's logic, not its timing
    try:
        occ = np.ones(24 ** 3)
        u = np.random.default_rng(1).standard_normal(3 * 25 ** 3)
        base = bench.cpu_baseline_matvec(occ, u, n=24, budget_s=0.5)
        assert base["kind"] == "port" and base["cores"] >= 1 and base["value"] > 0
    finally:
        bench.N_C2 = old
    _ = json
