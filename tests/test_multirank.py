"""Host-side logic of the N > 1 replica path (bench.py), exercised with the gloo backend on
CPU, world_size 2 (replicas only — the path has no exchange step)."""
import os
import socket

import pytest
import torch.multiprocessing as mp


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    port = s.getsockname()[1]
    s.close()
    return port


def _worker(rank, world, port, q):
    import torch.distributed as tdist
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    tdist.init_process_group("gloo", rank=rank, world_size=world)
    import bench
    my_ms = [120.0, 150.0][rank]          # rank 1 is the slow replica
    tot = bench.max_over_ranks(my_ms, "cpu")
    q.put((rank, tot, bench.replica_throughput(world, 5, tot)))
    tdist.barrier()
    tdist.destroy_process_group()


def test_max_over_ranks_and_replica_throughput_gloo():
    world = 2
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, world, port, q)) for r in range(world)]
    for p in procs:
        p.start()
    out = sorted(q.get(timeout=120) for _ in range(world))
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    for rank, tot, thr in out:
        assert tot == 150.0                               # every rank sees the max
        assert thr == pytest.approx(2 * 1000.0 * 5 / 150.0)


def test_dist_env_defaults(monkeypatch):
    import bench
    for k in ("RANK", "WORLD_SIZE", "LOCAL_RANK"):
        monkeypatch.delenv(k, raising=False)
    assert bench.dist_env() == (0, 1, 0)
