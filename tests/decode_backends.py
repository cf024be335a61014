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

    def __call__(self, x, out=None, accumulate=False, prologue=None, norm_weight=None, eps=1e-5):
        x = x.float()
        if prologue == "rmsnorm":
            x = x * torch.rsqrt(x.pow(2).mean(-1, keepdim=True) + eps) * norm_weight
        elif prologue == "rmsnorm_folded":  # the norm weight is already in the matrix
            x = x * torch.rsqrt(x.pow(2).mean(-1, keepdim=True) + eps)
        elif prologue == "swiglu":
            n = x.shape[-1] // 2
            x = torch.nn.functional.silu(x[..., :n]) * x[..., n:]
        if self.wd.device != x.device:
            self.wd = self.wd.to(x.device)
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

    @staticmethod
    def rope_kv(qkv, cos, sin, q_out, k_cache, v_cache, pos):
        B, H, ctx, hd = k_cache.shape
        q, k, v = qkv.view(B, 3, H, hd).unbind(1)
        half = hd // 2

        def rot(t):
            return torch.cat([t[..., :half] * cos - t[..., half:] * sin,
                              t[..., half:] * cos + t[..., :half] * sin], dim=-1)
        q_out.copy_(rot(q).view_as(q_out))
        k_cache[:, :, pos] = rot(k).to(k_cache.dtype)
        v_cache[:, :, pos] = v.to(v_cache.dtype)

    @classmethod
    def attention(cls, qkv, cos, sin, k_cache, v_cache, pos, scale, out, workspace):
        """RoPE + KV append, then torch SDPA over the f16 (or f32) cache."""
        B, H, ctx, hd = k_cache.shape
        q = torch.empty((B, H, 1, hd), dtype=k_cache.dtype, device=k_cache.device)
        cls.rope_kv(qkv, cos, sin, q, k_cache, v_cache, pos)
        att = torch.nn.functional.scaled_dot_product_attention(
            q.float(), k_cache[:, :, : pos + 1].float(), v_cache[:, :, : pos + 1].float(),
            scale=scale)
        out.copy_(att.reshape(B, H * hd))

    @staticmethod
    def attention_workspace(B, H, hd, ctx, device):
        return None

    @staticmethod
    def rmsnorm_f16(h, w, eps, out):
        out.copy_(h * torch.rsqrt(h.pow(2).mean(-1, keepdim=True) + eps) * w)
