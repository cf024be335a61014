"""Test-only linear backend for the decode driver: quantizes with the CPU
oracle (bit-exact with the reference) and multiplies with the dequantized
matrix on the CPU, so the tensor-parallel host logic can be checked with gloo
without a GPU.  Never used by the product path."""

import numpy as np
import torch

from oracle import qigen_oracle as orc


class OracleLinear:
    def __init__(self, w: torch.Tensor, qcfg):
        wn = w.detach().cpu().float().numpy()
        codes, s, z = orc.quantize_matrix(wn, qcfg.bits, qcfg.group_size)
        self.wd = torch.from_numpy(orc.dequantize_matrix(codes, s, z).astype(np.float64))
        self.K, self.N = wn.shape

    def __call__(self, x, out=None, accumulate=False):
        y = (x.double() @ self.wd).float()
        if out is None:
            return y
        if accumulate:
            out += y.view_as(out)
        else:
            out.copy_(y.view_as(out))
        return out

    @property
    def nbytes(self):
        return 0


class OracleBackend:
    linear = OracleLinear
