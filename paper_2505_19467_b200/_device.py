"""Device plumbing: CUDA availability, streams, host<->device staging.

PyTorch is used only to own device memory and streams; all arithmetic on
the step path happens in libkbe200.so.
"""

from __future__ import annotations

import numpy as np
import torch


def require_cuda() -> torch.device:
    if not torch.cuda.is_available():
        raise RuntimeError("kbe200 needs a CUDA device (B200, sm_100a); there is no CPU fallback")
    return torch.device("cuda", torch.cuda.current_device())


def stream_ptr(stream: torch.cuda.Stream | None = None) -> int:
    s = stream if stream is not None else torch.cuda.current_stream()
    return int(s.cuda_stream)


def as_device_c128(x, device=None) -> torch.Tensor:
    """Contiguous complex128 device tensor from numpy / torch input."""
    dev = device if device is not None else require_cuda()
    if isinstance(x, torch.Tensor):
        return x.to(device=dev, dtype=torch.complex128).contiguous()
    arr = np.ascontiguousarray(np.asarray(x, dtype=np.complex128))
    return torch.from_numpy(arr).to(dev)


def as_device_f64(x, device=None) -> torch.Tensor:
    dev = device if device is not None else require_cuda()
    if isinstance(x, torch.Tensor):
        return x.to(device=dev, dtype=torch.float64).contiguous()
    arr = np.ascontiguousarray(np.asarray(x, dtype=np.float64))
    return torch.from_numpy(arr).to(dev)


def ptr(t: torch.Tensor | None) -> int | None:
    return None if t is None else int(t.data_ptr())


def to_host(t: torch.Tensor) -> np.ndarray:
    return t.detach().cpu().numpy()
