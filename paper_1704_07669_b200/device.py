"""Device selection and numpy/torch plumbing (PyTorch is plumbing here:
device memory, streams and torch.distributed)."""

from __future__ import annotations

import numpy as np

from .errors import DeviceError


def torch_mod():
    import torch
    return torch


def default_device(device=None):
    """The CUDA device the product path runs on; raises without one (no CPU
    fallback exists for the sketch pass or the post-pass)."""
    torch = torch_mod()
    if not torch.cuda.is_available():
        raise DeviceError("no CUDA device visible: the sketch pass and post-pass run on the GPU only")
    if device is None:
        return torch.device("cuda", torch.cuda.current_device())
    dev = torch.device(device)
    if dev.type != "cuda":
        raise DeviceError(f"device must be a CUDA device, got {dev}")
    if dev.index is None:
        dev = torch.device("cuda", torch.cuda.current_device())
    return dev


def to_device64(x, device):
    """numpy / torch -> contiguous float64 CUDA tensor."""
    torch = torch_mod()
    if isinstance(x, torch.Tensor):
        return x.to(device=device, dtype=torch.float64).contiguous()
    return torch.as_tensor(np.ascontiguousarray(np.asarray(x, dtype=np.float64)), device=device)


def is_torch(x) -> bool:
    try:
        import torch
        return isinstance(x, torch.Tensor)
    except ImportError:  # pragma: no cover
        return False


def to_numpy(x) -> np.ndarray:
    if is_torch(x):
        return host_copy(x)
    return np.asarray(x)


def host_copy(t) -> np.ndarray:
    """CUDA tensor -> numpy through a page-locked staging tensor (torch's
    caching host allocator): a D2H copy at link speed instead of the
    pageable path's few GB/s. Host tensors pass through."""
    t = t.detach()
    if not t.is_cuda:
        return t.numpy()
    torch = torch_mod()
    out = torch.empty(t.shape, dtype=t.dtype, pin_memory=True)
    out.copy_(t, non_blocking=True)
    torch.cuda.current_stream(t.device).synchronize()
    return out.numpy()
