"""Device-memory plumbing (torch is used for allocation and streams only)."""

from __future__ import annotations

import numpy as np
import torch


def device() -> torch.device:
    if not torch.cuda.is_available():
        raise RuntimeError("paper_1909_07545_b200 needs a CUDA device (no CPU fallback)")
    return torch.device("cuda", torch.cuda.current_device())


def stream_ptr() -> int:
    return torch.cuda.current_stream().cuda_stream


def ptr(t: torch.Tensor | None) -> int | None:
    if t is None:
        return None
    assert t.is_cuda and t.is_contiguous()
    return t.data_ptr()


def empty(shape, dtype=torch.float32) -> torch.Tensor:
    return torch.empty(shape, dtype=dtype, device=device())


def zeros(shape, dtype=torch.float32) -> torch.Tensor:
    return torch.zeros(shape, dtype=dtype, device=device())


def upload(a, dtype=torch.float32) -> torch.Tensor:
    """Host array -> contiguous device tensor of `dtype` (bool masks -> uint8)."""
    if isinstance(a, torch.Tensor):
        t = a.to(device=device())
        if t.dtype == torch.bool:
            t = t.to(torch.uint8)
        return t.to(dtype).contiguous()
    arr = np.asarray(a)
    if arr.dtype == bool:
        arr = arr.astype(np.uint8)
    t = torch.from_numpy(np.ascontiguousarray(arr))
    return t.to(device=device(), dtype=dtype).contiguous()


def download(t: torch.Tensor, dtype=np.float64) -> np.ndarray:
    a = t.detach().cpu().numpy()
    if dtype is bool:
        return a.astype(bool)
    return a.astype(dtype)


def scratch(nbytes: int) -> torch.Tensor:
    return torch.empty(max(int(nbytes), 256), dtype=torch.uint8, device=device())
