"""Host-side logic of the multi-GPU path on CPU: world_size-2 `gloo` process
group. Frame partitioning covers a sequence exactly once, the job time is the
max over ranks, and the final gather reassembles every frame on rank 0. The
per-frame solve is a stub here (no GPU in this container); on GPUs it is
`solve_pyramid` and the backend is NCCL."""

import os
import socket

import numpy as np
import pytest
import torch.multiprocessing as mp


def test_partition_covers_sequence_once():
    from paper_1909_07545_b200.sequence import partition
    for n in (0, 1, 7, 256, 257):
        for world in (1, 2, 3, 4, 8):
            got = [i for r in range(world) for i in partition(n, world, r)]
            assert got == list(range(n))
            sizes = [len(partition(n, world, r)) for r in range(world)]
            assert max(sizes) - min(sizes) <= 1
    with pytest.raises(ValueError):
        partition(4, 2, 2)


def test_c4_rigs_vary_and_stay_valid():
    from paper_1909_07545_b200.sequence import c4_rig
    a, b = c4_rig(0), c4_rig(64)
    assert not np.allclose(a.pose.translation, b.pose.translation)
    for r in (a, b):
        R = r.pose.rotation
        assert np.allclose(R @ R.T, np.eye(3), atol=1e-12)


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    port = s.getsockname()[1]
    s.close()
    return port


def _worker(rank, world, port, n_frames, out_q):
    import torch.distributed as dist
    from paper_1909_07545_b200.sequence import (gather_results, max_over_ranks, partition,
                                                solve_block)
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        mine = partition(n_frames, world, rank)
        # stub solve: frame i -> constant map i (the GPU path runs solve_pyramid here)
        local = solve_block(((i, i) for i in mine), lambda i: np.full((4, 5), float(i)))
        t = max_over_ranks(0.1 * (rank + 1))
        frames = gather_results(local, rank, world, (4, 5))
        if rank == 0:
            out_q.put((t, sorted(frames), {k: float(v.mean()) for k, v in frames.items()}))
    finally:
        dist.destroy_process_group()


@pytest.mark.parametrize("n_frames", [5, 8])
def test_gloo_two_ranks_partition_time_and_gather(n_frames):
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, 2, port, n_frames, q)) for r in range(2)]
    for p in procs:
        p.start()
    t, frames, means = q.get(timeout=120)
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    assert abs(t - 0.2) < 1e-12                      # max over ranks
    assert frames == list(range(n_frames))           # every frame once
    assert all(means[i] == float(i) for i in frames)  # from the rank that owned it
