"""Host <-> device plumbing for the drop-in API (torch is plumbing only)."""

from __future__ import annotations

import numpy as np


def torch_mod():
    import torch

    return torch


def is_tensor(x) -> bool:
    try:
        import torch
    except ImportError:  # pragma: no cover
        return False
    return isinstance(x, torch.Tensor)


def to_device(x, pinned: bool = False):
    """Return (contiguous fp64 CUDA tensor, came_from_numpy)."""
    torch = torch_mod()
    if isinstance(x, torch.Tensor):
        t = x.to(device="cuda", dtype=torch.float64)
        return t.contiguous(), False
    a = np.ascontiguousarray(np.asarray(x, dtype=np.float64))
    h = torch.from_numpy(a)
    if pinned:
        h = h.pin_memory()
    return h.to("cuda", non_blocking=pinned), True


def to_host(t, as_numpy: bool):
    if as_numpy:
        return t.detach().cpu().numpy()
    return t


def empty(shape):
    torch = torch_mod()
    return torch.empty(tuple(shape), dtype=torch.float64, device="cuda")
