"""Group quantization on the GPU, bit-exact with the reference
(``qigen/quant.py``): same entry points, same fp64 parameter arithmetic
(quant.py:74-94), computed by ``qigen_quantize`` in libqigen_b200.

Arrays returned here are CUDA tensors (``CodeMatrix.numpy()`` copies to host).
"""

from __future__ import annotations

from dataclasses import dataclass

import numpy as np
import torch

from . import _dev
from ._lib import call
from .config import ConfigError, QuantConfig, ZeroMode, check_matrix_shape


@dataclass(frozen=True)
class GroupParams:
    """Scale and zero of one group (quant.py:26-31)."""

    scale: float
    zero: float


@dataclass
class CodeMatrix:
    """codes [n, m] u8 + scales/zeros [G, m] f32 (quant.py:34-67)."""

    codes: torch.Tensor
    scales: torch.Tensor
    zeros: torch.Tensor
    config: QuantConfig

    @property
    def n(self) -> int:
        return int(self.codes.shape[0])

    @property
    def m(self) -> int:
        return int(self.codes.shape[1])

    @property
    def groups(self) -> int:
        return int(self.scales.shape[0])

    def validate(self) -> None:
        g = self.config.groups_for_rows(self.n)
        if tuple(self.scales.shape) != (g, self.m) or tuple(self.zeros.shape) != (g, self.m):
            raise ConfigError(f"params shape {tuple(self.scales.shape)} does not match "
                              f"{g} groups x {self.m} columns")
        if self.codes.numel() and int(self.codes.max()) > self.config.max_code:
            raise ConfigError("codes exceed the bit-width mask")

    def numpy(self):
        return (_dev.to_host(self.codes), _dev.to_host(self.scales), _dev.to_host(self.zeros))


def quantize_matrix(w, config: QuantConfig) -> CodeMatrix:
    """quant.py:119-127 on the GPU.  ``w`` (n x m, numpy or torch) is converted
    to f32; non-finite values raise ConfigError like as_f32_matrix
    (config.py:123-132)."""
    wt = _dev.to_device(w, torch.float32)
    n, m = check_matrix_shape(wt.shape, "weight matrix")
    _dev.check_finite(wt, "weight matrix")
    G = config.groups_for_rows(n)
    codes = torch.empty((n, m), dtype=torch.uint8, device=wt.device)
    scales = torch.empty((G, m), dtype=torch.float32, device=wt.device)
    zeros = torch.empty((G, m), dtype=torch.float32, device=wt.device)
    call("qigen_quantize", wt.data_ptr(), n, m, config.bits, config.group_code,
         config.zero_mode.code, codes.data_ptr(), scales.data_ptr(), zeros.data_ptr(),
         _dev.stream_handle())
    return CodeMatrix(codes, scales, zeros, config)


def quantize_group(x, bits: int, zero_mode=ZeroMode.REAL32):
    """quant.py:97-108: one group -> (codes, GroupParams)."""
    v = _dev.to_device(x, torch.float32)
    if v.dim() != 1:
        raise ConfigError(f"group must be 1-D, got shape {tuple(v.shape)}")
    if v.numel() == 0:
        raise ConfigError("group must be non-empty")
    if bits not in (2, 3, 4):
        raise ConfigError(f"bits must be one of (2, 3, 4), got {bits}")
    cm = quantize_matrix(v[:, None], QuantConfig(bits, None, ZeroMode.coerce(zero_mode)))
    s, z = cm.scales.cpu(), cm.zeros.cpu()
    return cm.codes[:, 0], GroupParams(float(s[0, 0]), float(z[0, 0]))


def dequantize(codes, params: GroupParams):
    """quant.py:111-116: f32(s * (f32(c) - z))."""
    c = _dev.to_device(codes, torch.uint8).reshape(-1, 1)
    s = torch.tensor([[params.scale]], dtype=torch.float32, device=c.device)
    z = torch.tensor([[params.zero]], dtype=torch.float32, device=c.device)
    out = torch.empty(c.shape, dtype=torch.float32, device=c.device)
    call("qigen_dequantize", c.data_ptr(), s.data_ptr(), z.data_ptr(), c.shape[0], 1, 0,
         out.data_ptr(), _dev.stream_handle())
    return out[:, 0]


def dequantize_matrix(cm: CodeMatrix) -> torch.Tensor:
    """quant.py:130-138 on the GPU."""
    codes = _dev.to_device(cm.codes, torch.uint8)
    s = _dev.to_device(cm.scales, torch.float32)
    z = _dev.to_device(cm.zeros, torch.float32)
    n, m = codes.shape
    g = n // s.shape[0]
    out = torch.empty((n, m), dtype=torch.float32, device=codes.device)
    call("qigen_dequantize", codes.data_ptr(), s.data_ptr(), z.data_ptr(), n, m,
         0 if s.shape[0] == 1 else g, out.data_ptr(), _dev.stream_handle())
    return out


def codes_to_numpy(cm: CodeMatrix):
    return tuple(np.asarray(a) for a in cm.numpy())
