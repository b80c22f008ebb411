"""N > 1 is "replicas only": every rank runs its own solve and the job time is
the slowest rank.  This checks that reduction with the gloo backend, world_size 2, on CPU
(the NCCL run on GPUs uses the same helper)."""

import os
import socket

import pytest
import torch.multiprocessing as mp


def _free_port():
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        return s.getsockname()[1]


def _worker(rank, ws, port, out):
    import torch
    import torch.distributed as dist

    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=ws)
    try:
        import bench

        slow = bench.max_over_ranks(1.5 + rank, torch.device("cpu"), ws)
        out[rank] = slow
        # value = total steps of all ranks / slowest rank time
        out[ws + rank] = 100 * ws / slow
    finally:
        dist.destroy_process_group()


def test_max_over_ranks_gloo():
    ws = 2
    port = _free_port()
    out = mp.Manager().list([0.0] * (2 * ws))
    mp.spawn(_worker, args=(ws, port, out), nprocs=ws, join=True)
    assert list(out[:ws]) == [2.5, 2.5]
    assert out[ws] == pytest.approx(200 / 2.5)


def test_single_rank_passthrough():
    import bench

    assert bench.max_over_ranks(3.25, None, 1) == 3.25
