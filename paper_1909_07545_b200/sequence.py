"""Frame-parallel sequences across GPUs (BASELINE config 4).

Stereo frames are independent — `solve_pyramid` keeps no state between calls
(reference solver.py:401-452) — so a sequence is split into contiguous blocks
of frames, one block per rank (one process per GPU). The data path has no
collective; `gather_results` is the optional final gather to rank 0 (NCCL
over NVLink on GPUs, any torch.distributed backend in tests).
"""

from __future__ import annotations

import math

import numpy as np


def partition(n_frames: int, world: int, rank: int) -> range:
    """Contiguous block of frame indices owned by `rank` (sizes differ by <= 1)."""
    if world < 1 or not 0 <= rank < world or n_frames < 0:
        raise ValueError("bad partition request")
    base, extra = divmod(n_frames, world)
    start = rank * base + min(rank, extra)
    return range(start, start + base + (1 if rank < extra else 0))


def c4_pose(i: int, n_frames: int = 256):
    """Pose of frame i of the C4 sequence: C3's 6-DoF pose with a
    circular translation wobble and a periodic rotation scale."""
    from .camera import RelativePose
    t = np.array([0.08, 0.02, 0.03]) + 0.005 * np.array(
        [math.cos(2 * math.pi * i / n_frames), math.sin(2 * math.pi * i / n_frames), 0.0])
    rv = np.array([0.01, 0.03, -0.02]) * (1.0 + 0.1 * math.sin(2 * math.pi * i / 64))
    return RelativePose.from_displacement(t, rotvec=rv)


def c4_rig(i: int, n_frames: int = 256):
    """Rig of frame i of C4: the C3 unified 1024^2 camera pair at c4_pose(i)."""
    from .camera import StereoRig, UnifiedCamera
    cam = UnifiedCamera(width=1024, height=1024, fx=455.0, fy=455.0, cx=511.5, cy=511.5,
                        fov=math.pi, xi=0.9)
    return StereoRig(cam, cam, c4_pose(i, n_frames))


def solve_block(frames, solve_fn):
    """Solve this rank's frames in order: `frames` yields (index, payload),
    `solve_fn(payload) -> result`. Returns [(index, result)]."""
    return [(i, solve_fn(p)) for i, p in frames]


def max_over_ranks(seconds: float, device=None) -> float:
    """The job-level time of a step: the slowest rank's (torch.distributed MAX)."""
    import torch
    import torch.distributed as dist
    t = torch.tensor([float(seconds)], dtype=torch.float64, device=device)
    if dist.is_available() and dist.is_initialized() and dist.get_world_size() > 1:
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
    return float(t.item())


def gather_results(local: list, rank: int, world: int, shape, device=None):
    """Final gather of per-frame disparity maps to rank 0 (the only collective).

    `local` = [(frame index, (H, W) array)] of this rank. Returns on rank 0 a
    dict {frame index: array} covering every frame, None elsewhere.
    """
    import torch
    import torch.distributed as dist
    if world == 1:
        return {i: np.asarray(a) for i, a in local}
    counts = torch.tensor([len(local)], dtype=torch.int64, device=device)
    all_counts = [torch.zeros_like(counts) for _ in range(world)]
    dist.all_gather(all_counts, counts)
    cap = int(max(int(c.item()) for c in all_counts))
    buf = torch.zeros((cap, *shape), dtype=torch.float32, device=device)
    idx = torch.full((cap,), -1, dtype=torch.int64, device=device)
    for k, (i, a) in enumerate(local):
        buf[k] = torch.as_tensor(np.asarray(a, dtype=np.float32), device=device)
        idx[k] = i
    if rank == 0:
        bufs = [torch.zeros_like(buf) for _ in range(world)]
        idxs = [torch.zeros_like(idx) for _ in range(world)]
    else:
        bufs = idxs = None
    dist.gather(buf, bufs, dst=0)
    dist.gather(idx, idxs, dst=0)
    if rank != 0:
        return None
    out = {}
    for b, ix in zip(bufs, idxs):
        for k in range(cap):
            if int(ix[k]) >= 0:
                out[int(ix[k])] = b[k].cpu().numpy()
    return out
