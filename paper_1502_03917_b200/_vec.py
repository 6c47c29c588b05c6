"""Vector plumbing between the reference's numpy-array API and the device.

CUDA fp64 tensors pass through untouched (and are mutated in place where the
reference mutates); numpy arrays are copied to the device and the results
copied back, so reference-style callers work unchanged.
"""
from __future__ import annotations

import numpy as np


def as_device(x, n=None):
    import torch
    if isinstance(x, torch.Tensor):
        if not x.is_cuda:
            raise ValueError("expected a CUDA tensor (the device path has no "
                             "CPU fallback)")
        if x.dtype != torch.float64 or not x.is_contiguous():
            raise ValueError("expected a contiguous float64 CUDA tensor")
        if n is not None and x.shape != (n,):
            raise ValueError(f"vector has shape {tuple(x.shape)}, expected "
                             f"({n},)")
        return x, False
    a = np.ascontiguousarray(x, dtype=np.float64)
    if n is not None and a.shape != (n,):
        raise ValueError(f"vector has shape {a.shape}, expected ({n},)")
    return torch.from_numpy(a).to("cuda"), True


def back(t, was_np):
    return t.cpu().numpy() if was_np else t


def back_inplace(t, orig, was_np):
    if was_np:
        orig[...] = t.cpu().numpy()


def device_scalar():
    import torch
    return torch.empty(1, dtype=torch.float64, device="cuda")


def zeros(n):
    import torch
    return torch.zeros(n, dtype=torch.float64, device="cuda")
