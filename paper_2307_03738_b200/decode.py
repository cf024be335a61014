"""Tensor-parallel LLaMA-architecture decode driver over the quantized GEMV.

BASELINE configs[3] / [4] (north_star (d)): random-init LLaMA-7B (4-bit, g=128)
and LLaMA-65B (3-bit, g=64) decode steps, batch 1 (and 8 for 65B), fp16 KV
cache of 512 / 1024 past tokens, tensor-parallel over the GPUs of one node.
The reference has no model path; this driver is the consumer the
quantized GEMV exists for.

Sharding (Megatron pairing, one process per GPU, NCCL):
  * column-parallel, no communication: fused QKV (heads split across ranks) and
    fused gate|up (FFN columns split);
  * row-parallel: o_proj and down_proj take K-shards aligned to whole
    quantization groups and whole 256-row supersteps (uneven when the group
    count does not divide, e.g. 7B down_proj K = 11008 = 43 supersteps); rank 0
    accumulates the residual into its partial inside the GEMV epilogue, then
    one NCCL all-reduce per row-parallel layer (2 per layer);
  * lm_head is vocab-parallel (fp16), followed by an all-gather of logits.

Everything runs inside one CUDA graph per decode step.  The quantized linears
are ``PanelWeights`` (GPU quantize, bit-exact with quant.py, then the IMMA
GEMV).  A linear *backend* object builds them; tests inject a dequantized CPU
backend to check the TP logic with gloo (tests/test_decode_tp.py).
"""

from __future__ import annotations

import math
import os
from dataclasses import dataclass, replace

import torch
import torch.nn.functional as F

from . import _dev
from ._lib import call
from .config import QuantConfig
from .runtime import PanelWeights


@dataclass(frozen=True)
class LlamaConfig:
    n_layers: int
    d_model: int
    n_heads: int
    head_dim: int
    ffn: int
    vocab: int
    bits: int
    group: int | None
    norm_eps: float = 1e-5
    rope_theta: float = 10000.0

    @property
    def qcfg(self) -> QuantConfig:
        return QuantConfig(self.bits, self.group)


LLAMA_7B = LlamaConfig(32, 4096, 32, 128, 11008, 32000, 4, 128)
LLAMA_65B = LlamaConfig(80, 8192, 64, 128, 22016, 32000, 3, 64)


# ---------------------------------------------------------------------------
# shard arithmetic (pure; tested on CPU)
# ---------------------------------------------------------------------------

def even_split(total_units: int, world: int, rank: int) -> tuple[int, int]:
    """Units [lo, hi) of `rank` when `total_units` are spread as evenly as
    possible (the first `total_units % world` ranks get one more)."""
    base, extra = divmod(total_units, world)
    lo = rank * base + min(rank, extra)
    return lo, lo + base + (1 if rank < extra else 0)


def row_shard(K: int, group: int | None, world: int, rank: int) -> tuple[int, int]:
    """K-range of a row-parallel shard: whole groups and, when they fit, whole
    256-row supersteps of the GPU panel layout (uneven shards)."""
    if world == 1:
        return 0, K
    if group is None:
        raise ValueError("row-parallel sharding needs grouped quantization")
    unit = math.lcm(group, 256) if K % math.lcm(group, 256) == 0 else group
    if K % unit:
        raise ValueError(f"K={K} is not a multiple of the group size {group}")
    lo, hi = even_split(K // unit, world, rank)
    return lo * unit, hi * unit


def head_shard(n_heads: int, world: int, rank: int) -> tuple[int, int]:
    if n_heads % world:
        raise ValueError(f"{n_heads} heads do not split over {world} ranks")
    per = n_heads // world
    return rank * per, (rank + 1) * per


def col_shard(N: int, world: int, rank: int, align: int = 16) -> tuple[int, int]:
    """Output columns of a column-parallel shard (16-column panels)."""
    if N % align:
        return even_split(N, world, rank)
    lo, hi = even_split(N // align, world, rank)
    return lo * align, hi * align


# ---------------------------------------------------------------------------
# process group wrapper
# ---------------------------------------------------------------------------

class TP:
    """Rank/world of the tensor-parallel group (torch.distributed or single)."""

    def __init__(self, group=None):
        import torch.distributed as dist
        self.dist = dist if dist.is_available() and dist.is_initialized() else None
        self.group = group
        self.rank = self.dist.get_rank(group) if self.dist else 0
        self.world = self.dist.get_world_size(group) if self.dist else 1

    def all_reduce(self, t: torch.Tensor) -> torch.Tensor:
        if self.world > 1:
            self.dist.all_reduce(t, group=self.group)
        return t

    def all_gather_cat(self, t: torch.Tensor, sizes: list[int]) -> torch.Tensor:
        """Concatenate per-rank last-dim slices (uneven sizes padded)."""
        if self.world == 1:
            return t
        mx = max(sizes)
        pad = F.pad(t, (0, mx - t.shape[-1]))
        outs = [torch.empty_like(pad) for _ in range(self.world)]
        self.dist.all_gather(outs, pad.contiguous(), group=self.group)
        return torch.cat([o[..., :s] for o, s in zip(outs, sizes)], dim=-1)


class ShardTP(TP):
    """One rank's shard of a TP group of `world` ranks on a single GPU, with the
    collectives as no-ops: measures the per-GPU compute of a TP step (what the
    step costs before communication), e.g. to bound TP scaling on a one-GPU
    box.  Not for producing outputs."""

    def __init__(self, world: int, rank: int = 0):
        self.dist, self.group = None, None
        self.rank, self.world = rank, world

    def all_reduce(self, t: torch.Tensor) -> torch.Tensor:
        return t

    def all_gather_cat(self, t: torch.Tensor, sizes: list[int]) -> torch.Tensor:
        return F.pad(t, (0, sum(sizes) - t.shape[-1]))


# ---------------------------------------------------------------------------
# linear backends
# ---------------------------------------------------------------------------

class GpuLinear:
    """Quantized linear on the B200 GEMV: W [K, N] quantized on the GPU."""

    def __init__(self, w: torch.Tensor, qcfg: QuantConfig):
        self.pw = PanelWeights.from_float(w, qcfg)
        self.K, self.N = w.shape

    def __call__(self, x: torch.Tensor, out: torch.Tensor | None = None, accumulate: bool = False,
                 prologue: str | None = None, norm_weight=None, eps: float = 1e-5) -> torch.Tensor:
        return self.pw.gemv(x, out=out, accumulate=accumulate, prologue=prologue,
                            norm_weight=norm_weight, eps=eps)

    @property
    def nbytes(self) -> int:
        return self.pw.nbytes_algorithmic()


class GpuBackend:
    """The product backend: every op is a libqigen_b200 kernel (no fallback)."""

    linear = GpuLinear

    @staticmethod
    def rope_kv(qkv, cos, sin, q_out, k_cache, v_cache, pos):
        B, H, ctx, hd = k_cache.shape
        call("qigen_rope_kv", qkv.data_ptr(), B, H, hd, cos.data_ptr(), sin.data_ptr(),
             q_out.data_ptr(), k_cache.data_ptr(), v_cache.data_ptr(), ctx, pos,
             _dev.stream_handle())

    @staticmethod
    def attention(qkv, cos, sin, k_cache, v_cache, pos, scale, out, workspace):
        """RoPE + KV append + split-KV attention in one kernel (decode_ops.cu)."""
        B, H, ctx, hd = k_cache.shape
        call("qigen_attn_decode", qkv.data_ptr(), B, H, hd, cos.data_ptr(), sin.data_ptr(),
             k_cache.data_ptr(), v_cache.data_ptr(), ctx, pos, float(scale), out.data_ptr(),
             workspace.data_ptr(), workspace.numel(), _dev.stream_handle())

    @staticmethod
    def attention_workspace(B, H, hd, ctx, device):
        from ._lib import lib
        n = int(lib().qigen_attn_decode_workspace_size(B, H, hd, ctx))
        return torch.zeros(n, dtype=torch.uint8, device=device)

    @staticmethod
    def rmsnorm_f16(h, w, eps, out):
        call("qigen_rmsnorm_f16", h.data_ptr(), w.data_ptr(), h.shape[0], h.shape[1], float(eps),
             out.data_ptr(), _dev.stream_handle())


# ---------------------------------------------------------------------------
# the model
# ---------------------------------------------------------------------------

class LlamaTP:
    """One tensor-parallel shard of a random-init LLaMA-architecture model."""

    def __init__(self, cfg: LlamaConfig, *, batch: int = 1, max_ctx: int = 1024, seed: int = 0,
                 device=None, tp: TP | None = None, backend=GpuBackend,
                 kv_dtype=torch.float16):
        self.cfg, self.B, self.max_ctx = cfg, batch, max_ctx
        self.tp = tp or TP()
        self.dev = torch.device(device) if device is not None else torch.device("cuda")
        self.backend = backend
        r, w = self.tp.rank, self.tp.world
        d, hd = cfg.d_model, cfg.head_dim
        self.h0, self.h1 = head_shard(cfg.n_heads, w, r)
        self.nh = self.h1 - self.h0
        # FFN columns: also the K-shard of down_proj, so whole groups/supersteps
        self.f0, self.f1 = row_shard(cfg.ffn, cfg.group, w, r)
        self.nf = self.f1 - self.f0
        self.v_sizes = [col_shard(cfg.vocab, w, q)[1] - col_shard(cfg.vocab, w, q)[0]
                        for q in range(w)]
        self.v0, self.v1 = col_shard(cfg.vocab, w, r)
        # o_proj / down_proj K-shards: heads / FFN columns of this rank
        self.o_rows = (self.h0 * hd, self.h1 * hd)
        self.d_rows = (self.f0, self.f1)
        gen = torch.Generator(device=self.dev)

        def randn(shape, tag):
            gen.manual_seed(seed * 1_000_003 + tag)
            return torch.randn(shape, generator=gen, device=self.dev) * 0.02

        # off by default: neutral on 7B, slower on 65B (same-box A/B, bench.py)
        self.fold_qkv_norm = (batch <= 2 and backend is GpuBackend
                              and os.environ.get("QIGEN_FOLD_QKV_NORM", "0") == "1")
        self.layers = []
        for li in range(cfg.n_layers):
            base = 100 * li
            # column-parallel fused QKV: global W_q|W_k|W_v [d, 3 d]; this rank's heads
            wq, wk, wv = (randn((d, cfg.n_heads * hd), base + i) for i in range(3))
            sl = slice(self.h0 * hd, self.h1 * hd)
            n1 = torch.ones(d, device=self.dev)  # RMSNorm weights (random init: 1)
            n2 = torch.ones(d, device=self.dev)
            # option (QIGEN_FOLD_QKV_NORM=1, 1-2 tokens): fold the RMSNorm weight
            # into the QKV weights before quantization (diag(n1) W), so the GEMV
            # applies only 1/rms, in its epilogue, from the sums of squares of the
            # x chunks it already reads (no prep kernel)
            wqkv = torch.cat([wq[:, sl], wk[:, sl], wv[:, sl]], dim=1)
            if self.fold_qkv_norm:
                wqkv = wqkv * n1[:, None]
            wqkv = wqkv.contiguous()
            del wq, wk, wv
            wo = randn((cfg.n_heads * hd, d), base + 3)[self.o_rows[0]:self.o_rows[1]].contiguous()
            wg = randn((d, cfg.ffn), base + 4)[:, self.f0:self.f1]
            wu = randn((d, cfg.ffn), base + 5)[:, self.f0:self.f1]
            wgu = torch.cat([wg, wu], dim=1).contiguous()
            del wg, wu
            wd = randn((cfg.ffn, d), base + 6)[self.d_rows[0]:self.d_rows[1]].contiguous()
            layer = {
                "qkv": backend.linear(wqkv, cfg.qcfg),
                "o": backend.linear(wo, cfg.qcfg),
                "gu": backend.linear(wgu, cfg.qcfg),
                "down": backend.linear(wd, cfg.qcfg),
                "n1": n1,
                "n2": n2,
            }
            del wqkv, wo, wgu, wd
            self.layers.append(layer)
        self.norm = torch.ones(d, device=self.dev)
        gen.manual_seed(seed * 1_000_003 + 999_999)
        self.embed = (torch.randn((cfg.vocab, d), generator=gen, device=self.dev) * 0.02).half()
        gen.manual_seed(seed * 1_000_003 + 999_998)
        self.lm_head = (torch.randn((d, cfg.vocab), generator=gen, device=self.dev)
                        * 0.02)[:, self.v0:self.v1].half().t().contiguous()  # [V_l, d]
        # synthetic fp16 KV cache [layer][B, H_l, ctx, hd]: slices of one global
        # cache per layer, so every TP degree sees the same past tokens
        kshape = (cfg.n_layers, batch, self.nh, max_ctx, hd)
        self.k_cache = torch.empty(kshape, dtype=kv_dtype, device=self.dev)
        self.v_cache = torch.empty(kshape, dtype=kv_dtype, device=self.dev)
        for li in range(cfg.n_layers):
            for j, cache in enumerate((self.k_cache, self.v_cache)):
                g = randn((batch, cfg.n_heads, max_ctx, hd), 10_000_000 + 2 * li + j) * 50.0
                cache[li] = g[:, self.h0:self.h1].to(kv_dtype)
                del g
        self.attn_ws = backend.attention_workspace(batch, self.nh, hd, max_ctx, self.dev)
        inv = 1.0 / (cfg.rope_theta ** (torch.arange(0, hd, 2, device=self.dev).float() / hd))
        ang = torch.arange(max_ctx, device=self.dev).float()[:, None] * inv[None, :]
        self.cos, self.sin = ang.cos(), ang.sin()  # [ctx, hd/2]

    # -- accounting ---------------------------------------------------------
    def weight_bytes(self) -> int:
        """Algorithmic bytes of the quantized linears of this shard."""
        return sum(lay[k].nbytes for lay in self.layers for k in ("qkv", "o", "gu", "down"))

    def bytes_per_step(self, pos: int) -> int:
        """HBM bytes one decode step must read on this shard: quantized weights
        (codes + f32 scale/zero), fp16 lm_head shard, KV cache up to pos."""
        kv = 2 * self.cfg.n_layers * self.B * self.nh * (pos + 1) * self.cfg.head_dim * 2
        return self.weight_bytes() + self.lm_head.numel() * 2 + kv

    # -- one decode step ----------------------------------------------------
    def step(self, tokens: torch.Tensor, pos: int) -> torch.Tensor:
        """Greedy next tokens for `tokens` [B] at position `pos` (static shapes:
        graph-capturable for a fixed pos).  Per layer: QKV GEMV (RMSNorm fused:
        folded into W with 1/rms in the epilogue at 1-2 tokens, else a prologue)
        -> fused RoPE + KV append + attention -> o_proj GEMV (residual fused,
        all-reduce) -> gate|up GEMV (RMSNorm prologue) -> down GEMV (SwiGLU
        fused, residual fused, all-reduce)."""
        cfg, B, hd, be = self.cfg, self.B, self.cfg.head_dim, self.backend
        h = self.embed[tokens].float()                     # [B, d] residual stream
        cos, sin = self.cos[pos], self.sin[pos]
        scale = 1.0 / math.sqrt(hd)
        att = torch.empty((B, self.nh * hd), dtype=torch.float32, device=self.dev)
        for li, lay in enumerate(self.layers):
            if self.fold_qkv_norm:
                qkv = lay["qkv"](h, prologue="rmsnorm_folded", eps=cfg.norm_eps)
            else:
                qkv = lay["qkv"](h, prologue="rmsnorm", norm_weight=lay["n1"], eps=cfg.norm_eps)
            # RoPE + KV append + attention over positions 0..pos
            be.attention(qkv, cos, sin, self.k_cache[li], self.v_cache[li], pos, scale, att,
                         self.attn_ws)
            h = self._row_parallel(lay["o"], att, h)
            gu = lay["gu"](h, prologue="rmsnorm", norm_weight=lay["n2"], eps=cfg.norm_eps)
            h = self._row_parallel(lay["down"], gu, h, prologue="swiglu")
        xn = torch.empty((B, cfg.d_model), dtype=torch.float16, device=self.dev)
        be.rmsnorm_f16(h, self.norm, cfg.norm_eps, xn)
        logits = (xn @ self.lm_head.t()).float()           # [B, V_l]
        logits = self.tp.all_gather_cat(logits, self.v_sizes)
        self.last_logits = logits
        return logits.argmax(-1)

    def _row_parallel(self, lin, x: torch.Tensor, h: torch.Tensor, prologue=None) -> torch.Tensor:
        """Row-parallel linear + residual: rank 0 accumulates its partial into h
        inside the GEMV epilogue, the other ranks produce bare partials, and one
        all-reduce forms h + sum of partials on every rank."""
        if self.tp.rank == 0:
            lin(x, out=h, accumulate=True, prologue=prologue)
            out = h
        else:
            out = lin(x, prologue=prologue)
        return self.tp.all_reduce(out)


def shrink(cfg: LlamaConfig, **kw) -> LlamaConfig:
    return replace(cfg, **kw)
