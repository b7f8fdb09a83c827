"""Device-memory plumbing (PyTorch tensors as CUDA buffers).

PyTorch only allocates and moves memory here; every computation on the hot
path is a native kernel reached through the C-ABI.
"""

import numpy as np

_torch = None


def torch():
    global _torch
    if _torch is None:
        import torch as t
        _torch = t
    return _torch


def require_cuda(device: int = 0):
    t = torch()
    if not t.cuda.is_available():
        raise RuntimeError("the RIDC engine needs a CUDA device (no CPU fallback)")
    return t.device("cuda", device)


def to_device(a, device: int = 0):
    t = torch()
    arr = np.array(a, dtype=np.float64, copy=True)
    return t.from_numpy(arr).to(require_cuda(device))


def empty(n: int, device: int = 0):
    t = torch()
    return t.empty(int(n), dtype=t.float64, device=require_cuda(device))


def to_host(x) -> np.ndarray:
    return x.detach().cpu().numpy()
