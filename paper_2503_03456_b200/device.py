"""Device plumbing: column-major tensors, workspaces, streams (PyTorch is plumbing only).

Layout convention: a column-major m x n matrix with leading dimension m is
held in a contiguous torch tensor of shape (n, m) -- the row-major storage of
its transpose.  ``to_cm`` / ``from_cm`` convert numpy (C order) matrices.
"""

from __future__ import annotations

import numpy as np
import torch

from . import _native

_ws_cache: dict = {}


def device(dev=None) -> torch.device:
    if dev is None:
        if not torch.cuda.is_available():
            from .errors import DeviceError
            raise DeviceError("no CUDA device: the B200 solver has no CPU fallback")
        return torch.device("cuda", torch.cuda.current_device())
    return torch.device(dev)


def to_cm(M, dtype, dev) -> torch.Tensor:
    """numpy / torch (rows x cols) -> device tensor (cols, rows) == column-major M."""
    t = torch.as_tensor(np.asarray(M) if not isinstance(M, torch.Tensor) else M)
    return t.to(device=dev, dtype=dtype).t().contiguous()


def from_cm(t: torch.Tensor) -> np.ndarray:
    """device tensor (cols, rows) -> numpy (rows x cols)."""
    return t.t().cpu().numpy()


def workspace(nbytes: int, dev: torch.device) -> torch.Tensor:
    """Cached caller-owned workspace (the library never allocates)."""
    key = (dev.type, dev.index)
    buf = _ws_cache.get(key)
    if buf is None or buf.numel() < nbytes:
        buf = torch.empty(max(nbytes, 1), dtype=torch.uint8, device=dev)
        _ws_cache[key] = buf
    return buf


def stream_ptr(dev: torch.device) -> int:
    return torch.cuda.current_stream(dev).cuda_stream


def ptr(t: torch.Tensor) -> int:
    return t.data_ptr()


def dtype_code(t: torch.Tensor) -> int:
    return {torch.float32: 0, torch.float64: 1, torch.complex64: 2, torch.complex128: 3}[t.dtype]


def lib():
    return _native.lib()
