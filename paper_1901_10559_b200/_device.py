"""Device plumbing: torch owns device memory and streams; kernels come from
libidsketch_b200.so through _native.  Nothing here computes."""

import numpy as np
import torch

from . import _native


def device():
    if not torch.cuda.is_available():
        raise RuntimeError(
            "paper_1901_10559_b200 runs on a CUDA device (B200, sm_100a); "
            "there is no CPU fallback"
        )
    return torch.device("cuda", torch.cuda.current_device())


def stream_ptr():
    return ctypes_stream(torch.cuda.current_stream())


def ctypes_stream(stream):
    return int(stream.cuda_stream)


def ptr(t):
    """Device (or host) address of a tensor, or None."""
    return None if t is None else int(t.data_ptr())


def workspace(nbytes):
    return torch.empty(max(int(nbytes), 1), dtype=torch.uint8, device=device())


def empty(shape, dtype):
    return torch.empty(shape, dtype=dtype, device=device())


def zeros(shape, dtype):
    return torch.zeros(shape, dtype=dtype, device=device())


def to_device(x, dtype=None):
    """numpy array / CPU tensor / CUDA tensor -> CUDA tensor (no copy if already there)."""
    if isinstance(x, torch.Tensor):
        t = x
        if dtype is not None and t.dtype != dtype:
            t = t.to(dtype)
        if t.device.type != "cuda":
            t = t.to(device(), non_blocking=t.is_pinned())
        return t
    arr = np.asarray(x)
    t = torch.from_numpy(arr)
    if dtype is not None and t.dtype != dtype:
        t = t.to(dtype)
    return t.to(device())


def to_host(t):
    """Device tensor -> numpy through a pinned staging buffer (torch's
    caching host allocator reuses it): one DMA, no first-touch page faults
    of fresh pageable memory, one synchronization of the current stream."""
    t = t.detach()
    if t.device.type != "cuda":
        return t.numpy()
    h = torch.empty(t.shape, dtype=t.dtype, pin_memory=True)
    h.copy_(t, non_blocking=True)
    torch.cuda.current_stream().synchronize()
    return h.numpy()


def lib():
    return _native.load()
