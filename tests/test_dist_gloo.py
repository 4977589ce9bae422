"""Multi-process (world size 2, gloo, CPU) coverage of the N>1 bench path:
tasks sharded t % world == rank with no data-path collective, every task run
exactly once across ranks, and the max-over-ranks timing reduction."""

import json
import os
import socket

import numpy as np
import pytest
import torch.distributed as dist
import torch.multiprocessing as mp


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _worker(rank, world, port, out_dir):
    import torch

    import paper_1511_04348_b200 as tr

    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    rt = tr.Runtime(tr.homogeneous_machine(2), 4, mode="dryrun")
    m, k, n = 36, 20, 28  # 9 x 7 task grid, 5 k-steps
    _, s = rt.multiply(np.zeros((m, k)), np.zeros((k, n)), a_uid="A", b_uid="B", task_offset=rank,
                       task_stride=world)
    counts = torch.tensor([s.total_tasks, s.cache.input_requests, s.cache.writebacks], dtype=torch.int64)
    dist.all_reduce(counts, op=dist.ReduceOp.SUM)
    t = torch.tensor([float(rank + 1)], dtype=torch.float64)  # stand-in for the per-rank step time
    dist.all_reduce(t, op=dist.ReduceOp.MAX)
    with open(os.path.join(out_dir, f"r{rank}.json"), "w") as f:
        json.dump({"counts": counts.tolist(), "tmax": float(t.item()), "mine": s.total_tasks}, f)
    dist.barrier()
    dist.destroy_process_group()


@pytest.mark.timeout(180)
def test_two_rank_task_sharding(tmp_path):
    world = 2
    mp.start_processes(_worker, args=(world, _free_port(), str(tmp_path)), nprocs=world, join=True,
                       start_method="spawn")
    res = [json.loads((tmp_path / f"r{r}.json").read_text()) for r in range(world)]
    for r in res:
        total, requests, writebacks = r["counts"]
        assert total == 9 * 7  # every task exactly once across the two ranks
        assert requests == 2 * 63 * 5 and writebacks == 63
        assert r["tmax"] == 2.0
    assert [r["mine"] for r in res] == [32, 31]


def _bench_worker(rank, world, port, out_dir):
    """bench.py's torchrun plumbing: rank 0 alone drives the N-GPU machine (here a
    dry-run machine of N logical devices), the other ranks only join the max."""
    import sys
    from pathlib import Path

    sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
    import bench
    import paper_1511_04348_b200 as tr

    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    coord = bench.Coordinator(env={"WORLD_SIZE": str(world), "RANK": str(rank)})
    args = bench.parse(["--gpus", "1"])
    ng = bench.n_gpus_for(args, coord.world)
    t_local, tasks = 0.0, None
    if coord.rank == 0:
        with tr.Runtime(tr.homogeneous_machine(ng), 4, mode="dryrun") as rt:
            _, s = rt.multiply(np.zeros((36, 20)), np.zeros((20, 28)), a_uid="A", b_uid="B")
        tasks = s.tasks_by_device
        t_local = 2.5
    t = coord.max_over_ranks(t_local)
    coord.close()
    with open(os.path.join(out_dir, f"b{rank}.json"), "w") as f:
        json.dump({"ng": ng, "t": t, "tasks": tasks}, f)


@pytest.mark.timeout(180)
def test_bench_one_process_drives_all_gpus(tmp_path):
    world = 2
    mp.start_processes(_bench_worker, args=(world, _free_port(), str(tmp_path)), nprocs=world, join=True,
                       start_method="spawn")
    r0, r1 = (json.loads((tmp_path / f"b{r}.json").read_text()) for r in range(world))
    assert r0["ng"] == r1["ng"] == 2  # --gpus 1 under WORLD_SIZE=2: one process, two GPUs
    assert r0["t"] == r1["t"] == 2.5  # max over ranks; rank 1 did no work
    assert r1["tasks"] is None and sum(r0["tasks"].values()) == 9 * 7 and len(r0["tasks"]) == 2
