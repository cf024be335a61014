"""Device-memory plumbing (torch is used for allocation and streams only)."""

from __future__ import annotations

import numpy as np
import torch

from .config import ConfigError


def require_cuda() -> torch.device:
    if not torch.cuda.is_available():
        raise RuntimeError("qigen-b200 needs a CUDA device (B200, sm_100a); "
                           "there is no CPU fallback")
    return torch.device("cuda", torch.cuda.current_device())


def stream_handle() -> int:
    return torch.cuda.current_stream().cuda_stream


def to_device(arr, dtype: torch.dtype) -> torch.Tensor:
    """numpy array / torch tensor / sequence -> contiguous CUDA tensor."""
    dev = require_cuda()
    if isinstance(arr, torch.Tensor):
        t = arr
    else:
        a = np.asarray(arr)
        t = torch.from_numpy(np.ascontiguousarray(a))
    return t.to(device=dev, dtype=dtype).contiguous()


def is_host(arr) -> bool:
    return not (isinstance(arr, torch.Tensor) and arr.is_cuda)


def to_host(t: torch.Tensor) -> np.ndarray:
    return t.detach().cpu().numpy()


def check_finite(t: torch.Tensor, name: str) -> None:
    if not bool(torch.isfinite(t).all()):
        raise ConfigError(f"{name} contains non-finite values")


def ptr(t: torch.Tensor | None) -> int | None:
    return None if t is None else t.data_ptr()
