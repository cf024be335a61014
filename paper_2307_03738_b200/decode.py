"""Tensor-parallel LLaMA-architecture decode driver over the quantized GEMV.

BASELINE configs[3] / [4] (north_star (d)): random-init LLaMA-7B (4-bit, g=128)
and LLaMA-65B (3-bit, g=64) decode steps, batch 1 (and 8 for 65B), fp16 KV
cache of 512 / 1024 past tokens, tensor-parallel over the GPUs of one node.
The reference has no model path; this driver is the consumer the
quantized GEMV exists for.

Sharding (Megatron pairing, one process per GPU):
  * column-parallel, no communication: fused QKV (heads split across ranks) and
    fused gate|up (FFN columns split);
  * row-parallel: o_proj and down_proj take K-shards aligned to whole
    quantization groups and whole 256-row supersteps (uneven when the group
    count does not divide, e.g. 7B down_proj K = 11008 = 43 supersteps).  The
    all-reduce after each (2 per layer) is the one-shot push of csrc/tp.cuh:
    the GEMV epilogue stores its partial into every rank's inbox over NVLink
    (CUDA IPC), then a reduce kernel adds the partials to the residual in rank
    order ("push").  Without peer mappings it falls back
    to rank 0 accumulating the residual in its GEMV epilogue + an NCCL
    all-reduce ("nccl");
  * lm_head is vocab-parallel (fp16) with the RMSNorm and the greedy argmax
    fused into one kernel per rank (csrc/lmhead.cu); ranks exchange only
    (max, index) pairs.

The step is a generator of phases (``step_phases``) that yields where a rank
needs the other ranks' data; ``step`` runs it to the end.  Several ranks can
therefore be emulated on ONE GPU (``emulated_tp``): every rank's phase k is
issued before any rank's phase k+1, so no kernel waits on one that has not
been launched before it (B200_PROFILING.md: ranks that wait on one another
must not run as separate launches unless their order guarantees progress).

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
        self._post = None

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

    # greedy token across vocab shards: each rank posts (max, global index) per
    # token, the token is the first rank's index among the maxima (= the lowest
    # global index, torch.argmax's tie rule over the concatenated logits)
    def argmax_post(self, mx: torch.Tensor, ix: torch.Tensor, logits=None, sizes=None) -> None:
        self._post = (mx, ix, logits, sizes)

    def argmax_collect(self):
        mx, ix, logits, sizes = self._post
        self._post = None
        if self.world == 1:
            return ix, logits
        pair = torch.stack([mx.double(), ix.double()], dim=-1)  # [B, 2]
        outs = [torch.empty_like(pair) for _ in range(self.world)]
        self.dist.all_gather(outs, pair, group=self.group)
        full = None if logits is None else self.all_gather_cat(logits, sizes)
        return pick_argmax(torch.stack(outs)), full


def pick_argmax(pairs: torch.Tensor) -> torch.Tensor:
    """pairs [world, B, 2] of (max, global index) -> global argmax per token."""
    r = pairs[..., 0].argmax(0)  # first maximal rank
    return pairs[r, torch.arange(pairs.shape[1], device=pairs.device), 1].long()


class ShardTP(TP):
    """One rank's shard of a TP group of `world` ranks on a single GPU, with the
    collectives as no-ops: measures the per-GPU compute of a TP step (what the
    step costs before communication), e.g. to bound TP scaling on a one-GPU
    box.  Not for producing outputs."""

    def __init__(self, world: int, rank: int = 0):
        self.dist, self.group = None, None
        self.rank, self.world = rank, world
        self._post = None

    def all_reduce(self, t: torch.Tensor) -> torch.Tensor:
        return t

    def all_gather_cat(self, t: torch.Tensor, sizes: list[int]) -> torch.Tensor:
        return F.pad(t, (0, sum(sizes) - t.shape[-1]))

    def argmax_collect(self):
        mx, ix, logits, sizes = self._post
        self._post = None
        return ix, None if logits is None else self.all_gather_cat(logits, sizes)


class EmuGroup:
    """A TP group of `world` ranks emulated in one process on one GPU: the
    (max, index) / logit exchange goes through shared tensors; the row-parallel
    all-reduces must use the push comm (TpComm.emulated)."""

    def __init__(self, world: int):
        self.world = world
        self.posts = [None] * world


class EmuTP(TP):
    def __init__(self, group: EmuGroup, rank: int):
        self.dist, self.group = None, group
        self.rank, self.world = rank, group.world
        self._post = None

    def all_reduce(self, t):
        raise RuntimeError("emulated TP ranks all-reduce through the push comm only")

    def all_gather_cat(self, t, sizes):
        raise RuntimeError("emulated TP ranks exchange through argmax_post / argmax_collect")

    def argmax_post(self, mx, ix, logits=None, sizes=None) -> None:
        self.group.posts[self.rank] = (mx, ix, logits)

    def argmax_collect(self):
        posts = self.group.posts
        pairs = torch.stack([torch.stack([p[0].double(), p[1].double()], dim=-1) for p in posts])
        full = None
        if all(p[2] is not None for p in posts):
            full = torch.cat([p[2] for p in posts], dim=-1)
        return pick_argmax(pairs), full


class TpComm:
    """The push all-reduce of csrc/tp.cuh for one rank: its buffer, the peers'
    buffers mapped into this process, and the C handle."""

    def __init__(self, rank, world, d, bmax, layers, bases, owned=(), opened=()):
        import ctypes
        from ._lib import lib
        self.rank, self.world, self.d, self.bmax = rank, world, d, bmax
        self._owned, self._opened = list(owned), list(opened)
        arr = (ctypes.c_void_p * 8)(*[ctypes.c_void_p(b) for b in bases])
        h = ctypes.c_void_p()
        call("qigen_tp_create", rank, world, d, bmax, layers, arr, ctypes.byref(h))
        self._h = h
        self._lib = lib()

    @staticmethod
    def _alloc(world, d, bmax, with_handle):
        import ctypes
        from ._lib import lib
        nbytes = int(lib().qigen_tp_buffer_size(world, d, bmax))
        p = ctypes.c_void_p()
        hbuf = ctypes.create_string_buffer(64) if with_handle else None
        call("qigen_tp_alloc", nbytes, ctypes.byref(p), hbuf)
        return p.value, (hbuf.raw if with_handle else None)

    @classmethod
    def setup_dist(cls, tp: TP, d, bmax, layers) -> "TpComm":
        """Real ranks (one process per GPU): allocate, exchange CUDA IPC handles
        over the process group, map every peer's buffer."""
        import ctypes
        base, handle = cls._alloc(tp.world, d, bmax, True)
        handles = [None] * tp.world
        tp.dist.all_gather_object(handles, handle, group=tp.group)
        bases, opened = [], []
        for q, hq in enumerate(handles):
            if q == tp.rank:
                bases.append(base)
                continue
            p = ctypes.c_void_p()
            call("qigen_tp_open_peer", ctypes.create_string_buffer(hq, 64), ctypes.byref(p))
            bases.append(p.value)
            opened.append(p.value)
        tp.dist.barrier(group=tp.group)
        return cls(tp.rank, tp.world, d, bmax, layers, bases, owned=[base], opened=opened)

    @classmethod
    def emulated(cls, world, d, bmax, layers) -> list["TpComm"]:
        """`world` ranks on this GPU: plain device buffers, each rank's peers are
        the other ranks' buffers."""
        bases = [cls._alloc(world, d, bmax, False)[0] for _ in range(world)]
        comms = [cls(r, world, d, bmax, layers, bases) for r in range(world)]
        comms[0]._owned = bases
        return comms

    def step_begin(self) -> None:
        call("qigen_tp_step_begin", self._h, _dev.stream_handle())

    def reduce(self, slot: int, layer: int, h: torch.Tensor) -> None:
        call("qigen_tp_reduce", self._h, slot, layer, h.data_ptr(), h.shape[0],
             _dev.stream_handle())

    def error(self) -> int:
        import ctypes
        v = ctypes.c_int()
        call("qigen_tp_error", self._h, ctypes.byref(v))
        return v.value

    def __del__(self):
        try:
            lib_ = self._lib
            for p in getattr(self, "_opened", []):
                lib_.qigen_tp_close_peer(p)
            for p in getattr(self, "_owned", []):
                lib_.qigen_tp_free(p)
            if getattr(self, "_h", None):
                lib_.qigen_tp_destroy(self._h)
        except Exception:  # noqa: BLE001
            pass


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

    def chain(self, x, out, **kw):
        """A GEMV of the dependent decode chain (PanelWeights.chain)."""
        return self.pw.chain(x, out, **kw)

    def push(self, comm: "TpComm", slot: int, x: torch.Tensor, prologue: str | None = None):
        """Row-parallel partial x W into every rank's inbox (qigen_gemv_tp_push)."""
        self.pw.push(comm, slot, x, prologue=prologue)

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
    def attention(qkv, cos, sin, k_cache, v_cache, pos, scale, out, workspace, o_digits=None,
                  o_group=None):
        """RoPE + KV append + split-KV attention in one kernel (decode_ops.cu);
        with ``o_digits`` the heads also write the o_proj GEMV's activation
        digits (qigen_attn_decode_chain)."""
        B, H, ctx, hd = k_cache.shape
        if o_digits is None:
            call("qigen_attn_decode", qkv.data_ptr(), B, H, hd, cos.data_ptr(), sin.data_ptr(),
                 k_cache.data_ptr(), v_cache.data_ptr(), ctx, pos, float(scale), out.data_ptr(),
                 workspace.data_ptr(), workspace.numel(), _dev.stream_handle())
        else:
            call("qigen_attn_decode_chain", qkv.data_ptr(), B, H, hd, cos.data_ptr(),
                 sin.data_ptr(), k_cache.data_ptr(), v_cache.data_ptr(), ctx, pos, float(scale),
                 out.data_ptr(), workspace.data_ptr(), workspace.numel(), o_digits.data_ptr(),
                 0 if o_group is None else int(o_group), _dev.stream_handle())

    @staticmethod
    def attention_workspace(B, H, hd, ctx, device):
        from ._lib import lib
        n = int(lib().qigen_attn_decode_workspace_size(B, H, hd, ctx))
        return torch.zeros(n, dtype=torch.uint8, device=device)

    @staticmethod
    def rmsnorm_f16(h, w, eps, out):
        call("qigen_rmsnorm_f16", h.data_ptr(), w.data_ptr(), h.shape[0], h.shape[1], float(eps),
             out.data_ptr(), _dev.stream_handle())

    @staticmethod
    def lm_head_workspace(V, d, B, device):
        from ._lib import lib
        n = int(lib().qigen_lm_head_workspace_size(V, d, B))
        return torch.zeros(n, dtype=torch.uint8, device=device)

    @staticmethod
    def lm_head(h, norm_w, eps, w_f16, v0, logits, mx, ix, workspace):
        """Final RMSNorm + fp16 vocab-shard GEMV + greedy argmax, one kernel
        (csrc/lmhead.cu): mx / ix get each token's max logit and global index."""
        call("qigen_lm_head", h.data_ptr(), norm_w.data_ptr(), float(eps), w_f16.data_ptr(),
             w_f16.shape[0], w_f16.shape[1], h.shape[0], int(v0),
             None if logits is None else logits.data_ptr(), mx.data_ptr(), ix.data_ptr(),
             workspace.data_ptr(), workspace.numel(), _dev.stream_handle())


# ---------------------------------------------------------------------------
# the model
# ---------------------------------------------------------------------------

class LlamaTP:
    """One tensor-parallel shard of a random-init LLaMA-architecture model.

    ``comm``: how the row-parallel all-reduces run when world > 1 —
    ``"auto"`` (the push comm over CUDA IPC when the backend is the GPU one and
    the peers map, else NCCL), ``"push"``, ``"nccl"``, or a ``TpComm`` (emulated
    ranks).  ``keep_logits``: also assemble the full logits (``last_logits``)."""

    def __init__(self, cfg: LlamaConfig, *, batch: int = 1, max_ctx: int = 1024, seed: int = 0,
                 device=None, tp: TP | None = None, backend=GpuBackend,
                 kv_dtype=torch.float16, comm="auto", keep_logits: bool = True,
                 stack: bool | None = None):
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
        # one GPU, 1-2 tokens: o_proj and down write the activation digits of the
        # next RMSNorm'd GEMV (gate|up, next layer's QKV) in their epilogue, the
        # norm folded (1 / rms in the consumer's epilogue), so those GEMVs need no
        # prep kernel or prologue (qigen_gemv_chain).  Measured (same box, B200,
        # 7B TP1 B=1): 625 vs 591 tok/s; letting gate|up also write SwiGLU digits
        # for down (256-column CTAs) measured slower (554) and was dropped.
        self.chained = (self.tp.world == 1 and backend is GpuBackend and not self.fold_qkv_norm
                        and batch <= 2 and os.environ.get("QIGEN_CHAIN", "1") == "1")
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
        self.keep_logits = keep_logits
        if self.chained:
            from .runtime import digits_buffer, ss_count
            self.dig = [digits_buffer(d, batch, self.dev) for _ in range(2)]
            # attention -> o_proj digits (head_dim 128, o_proj group >= 64)
            self.att_dig = (digits_buffer(self.nh * hd, batch, self.dev)
                            if hd == 128 and (cfg.group is None or cfg.group >= 64) else None)
            self.ssc = ss_count(d)
            self.ss = [torch.zeros(batch * self.ssc, device=self.dev) for _ in range(2)]
        # one GPU, one token: all layers as ONE persistent launch (csrc/decode_stack.cu);
        # shapes outside its limits keep the per-op chain above
        self.stack, self.stack_reason = None, "not requested"
        if stack is None:
            stack = os.environ.get("QIGEN_STACK", "1") == "1"
        if (stack and self.tp.world == 1 and backend is GpuBackend and batch == 1
                and kv_dtype == torch.float16):
            self.stack = self._make_stack()
        self.fused_head = hasattr(backend, "lm_head") and self.dev.type == "cuda" and batch <= 8
        if self.fused_head:
            self.head_ws = backend.lm_head_workspace(self.v1 - self.v0, d, batch, self.dev)
        # row-parallel all-reduce: the push comm (csrc/tp.cuh) or NCCL
        self.comm, self.comm_kind = None, None
        if self.tp.world > 1:
            if isinstance(comm, TpComm):
                self.comm, self.comm_kind = comm, "push (emulated ranks)"
            elif comm in ("auto", "push") and backend is GpuBackend and self.tp.dist is not None:
                try:
                    self.comm = TpComm.setup_dist(self.tp, d, batch, cfg.n_layers)
                    self.comm_kind = "push (one-shot, GEMV epilogue -> peer inboxes over NVLink)"
                except Exception as e:  # noqa: BLE001
                    if comm == "push":
                        raise
                    self.comm_kind = f"nccl (push setup failed: {type(e).__name__})"
            else:
                self.comm_kind = "nccl"
        inv = 1.0 / (cfg.rope_theta ** (torch.arange(0, hd, 2, device=self.dev).float() / hd))
        ang = torch.arange(max_ctx, device=self.dev).float()[:, None] * inv[None, :]
        self.cos, self.sin = ang.cos(), ang.sin()  # [ctx, hd/2]

    def _make_stack(self):
        """The persistent decode-stack handle over this model's weights and KV
        caches, or None where the kernel does not take the shape."""
        import ctypes
        from ._lib import StackDesc, StackLayer, UnsupportedError
        cfg = self.cfg
        if cfg.group is None:
            return None
        desc = StackDesc(cfg.n_layers, cfg.d_model, cfg.n_heads, cfg.head_dim, cfg.ffn, cfg.bits,
                         cfg.group, self.max_ctx, cfg.norm_eps)
        arr = (StackLayer * cfg.n_layers)()
        for li, lay in enumerate(self.layers):
            for j, k in enumerate(("qkv", "o", "gu", "down")):
                arr[li].qw[j] = lay[k].pw.qw.data_ptr()
                arr[li].qsz[j] = lay[k].pw.qsz.data_ptr()
            arr[li].norm1, arr[li].norm2 = lay["n1"].data_ptr(), lay["n2"].data_ptr()
            arr[li].k_cache = self.k_cache[li].data_ptr()
            arr[li].v_cache = self.v_cache[li].data_ptr()
        h = ctypes.c_void_p()
        try:
            call("qigen_decode_stack_create", ctypes.byref(desc), arr, ctypes.byref(h))
        except UnsupportedError as e:
            self.stack_reason = str(e)
            return None
        return h

    def stack_error(self) -> int:
        """Non-zero if a wait inside the persistent kernel timed out (synchronises)."""
        import ctypes
        v = ctypes.c_int()
        call("qigen_decode_stack_error", self.stack, ctypes.byref(v))
        return v.value

    def __del__(self):
        try:
            if getattr(self, "stack", None):
                from ._lib import lib
                lib().qigen_decode_stack_destroy(self.stack)
        except Exception:  # noqa: BLE001
            pass

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
        graph-capturable for a fixed pos)."""
        for _ in self.step_phases(tokens, pos):
            pass
        return self.next_tokens

    def step_phases(self, tokens: torch.Tensor, pos: int):
        """The decode step as phases; yields where the other ranks' data is
        needed next.  Per layer: QKV GEMV (RMSNorm fused: folded into W with
        1/rms in the epilogue at 1-2 tokens, else a prologue) -> fused RoPE + KV
        append + attention -> o_proj GEMV (+ all-reduce with the residual) ->
        gate|up GEMV (RMSNorm prologue) -> down GEMV (SwiGLU prologue, +
        all-reduce with the residual); then the fused final RMSNorm + LM head +
        argmax."""
        cfg, B, hd, be = self.cfg, self.B, self.cfg.head_dim, self.backend
        h = self.embed[tokens].float()                     # [B, d] residual stream
        if self.comm is not None:
            self.comm.step_begin()
        cos, sin = self.cos[pos], self.sin[pos]
        scale = 1.0 / math.sqrt(hd)
        att = torch.empty((B, self.nh * hd), dtype=torch.float32, device=self.dev)
        if self.stack is not None:  # every layer in one persistent launch
            h_out = torch.empty_like(h)
            call("qigen_decode_stack_run", self.stack, h.data_ptr(), h_out.data_ptr(),
                 cos.data_ptr(), sin.data_ptr(), pos, float(scale), _dev.stream_handle())
            h = h_out
        for li, lay in enumerate(self.layers if self.stack is None else ()):
            if self.chained:
                yield from self._layer_chained(li, lay, h, att, cos, sin, pos, scale)
                continue
            if self.fold_qkv_norm:
                qkv = lay["qkv"](h, prologue="rmsnorm_folded", eps=cfg.norm_eps)
            else:
                qkv = lay["qkv"](h, prologue="rmsnorm", norm_weight=lay["n1"], eps=cfg.norm_eps)
            # RoPE + KV append + attention over positions 0..pos
            be.attention(qkv, cos, sin, self.k_cache[li], self.v_cache[li], pos, scale, att,
                         self.attn_ws)
            yield from self._row_parallel(lay["o"], att, h, None, 0, li)
            gu = lay["gu"](h, prologue="rmsnorm", norm_weight=lay["n2"], eps=cfg.norm_eps)
            yield from self._row_parallel(lay["down"], gu, h, "swiglu", 1, li)
        Vl = self.v1 - self.v0
        if self.fused_head:
            logits = (torch.empty((B, Vl), dtype=torch.float32, device=self.dev)
                      if self.keep_logits else None)
            mx = torch.empty(B, dtype=torch.float32, device=self.dev)
            ix = torch.empty(B, dtype=torch.int64, device=self.dev)
            be.lm_head(h, self.norm, cfg.norm_eps, self.lm_head, self.v0, logits, mx, ix,
                       self.head_ws)
        else:
            xn = torch.empty((B, cfg.d_model), dtype=torch.float16, device=self.dev)
            be.rmsnorm_f16(h, self.norm, cfg.norm_eps, xn)
            logits = (xn.double() @ self.lm_head.double().t()).float()   # [B, V_l]
            mx, ix = logits.max(-1)
            ix = ix + self.v0
        self.tp.argmax_post(mx, ix, logits if self.keep_logits else None, self.v_sizes)
        yield
        self.next_tokens, self.last_logits = self.tp.argmax_collect()

    def _layer_chained(self, li, lay, h, att, cos, sin, pos, scale):
        """One layer on one GPU without activation prep kernels: o_proj and down
        write the activation digits of gate|up and of the next layer's QKV
        (times that GEMV's RMSNorm weight) plus their sums of squares, the
        consumers apply 1 / rms in their epilogue."""
        cfg, B, hd = self.cfg, self.B, self.cfg.head_dim
        eps, g = cfg.norm_eps, cfg.group
        qkv = torch.empty((B, 3 * self.nh * hd), dtype=torch.float32, device=self.dev)
        if li == 0:  # the embedding has no producer GEMV
            lay["qkv"](h, out=qkv, prologue="rmsnorm", norm_weight=lay["n1"], eps=eps)
        else:
            lay["qkv"].chain(None, qkv, tokens=B, digits_in=self.dig[1], ss_in=self.ss[1],
                             ss_count=self.ssc, eps=eps)
        self.backend.attention(qkv, cos, sin, self.k_cache[li], self.v_cache[li], pos, scale,
                               att, self.attn_ws, o_digits=self.att_dig, o_group=g)
        lay["o"].chain(att, h, tokens=B, accumulate=True, digits_in=self.att_dig,
                       digits_out=self.dig[0], out_scale=lay["n2"], out_group=g,
                       ss_out=self.ss[0])
        gu = torch.empty((B, 2 * self.nf), dtype=torch.float32, device=self.dev)
        lay["gu"].chain(None, gu, tokens=B, digits_in=self.dig[0], ss_in=self.ss[0],
                        ss_count=self.ssc, eps=eps)
        last = li + 1 == len(self.layers)
        lay["down"].chain(gu, h, tokens=B, accumulate=True, prologue="swiglu",
                          digits_out=None if last else self.dig[1],
                          out_scale=None if last else self.layers[li + 1]["n1"], out_group=g,
                          ss_out=None if last else self.ss[1])
        return
        yield  # (generator)

    def _row_parallel(self, lin, x: torch.Tensor, h: torch.Tensor, prologue, slot: int,
                      layer: int):
        """Row-parallel linear + residual, h updated in place.  World 1: the GEMV
        adds its output to h in its epilogue.  Push comm: every rank's GEMV
        stores its partial into every rank's inbox, then (after the phase
        boundary) each rank adds the partials to h in rank order.  NCCL: rank 0
        accumulates into h, the others produce bare partials, one all-reduce."""
        if self.tp.world == 1:
            lin(x, out=h, accumulate=True, prologue=prologue)
            return
        if self.comm is not None:
            lin.push(self.comm, slot, x, prologue=prologue)
            yield
            self.comm.reduce(slot, layer, h)
            return
        if self.tp.rank == 0:
            lin(x, out=h, accumulate=True, prologue=prologue)
            self.tp.all_reduce(h)
        else:
            h.copy_(self.tp.all_reduce(lin(x, prologue=prologue)))
        return
        yield  # (generator)


def emulated_tp(cfg: LlamaConfig, world: int, **kw) -> list[LlamaTP]:
    """`world` TP ranks of one model on THIS GPU (for tests and per-rank
    measurements): one LlamaTP shard per rank, the push comm over plain device
    buffers.  Drive them with ``emulated_step``."""
    group = EmuGroup(world)
    comms = TpComm.emulated(world, cfg.d_model, kw.get("batch", 1), cfg.n_layers)
    return [LlamaTP(cfg, tp=EmuTP(group, r), comm=comms[r], **kw) for r in range(world)]


def emulated_step(models: list[LlamaTP], tokens: torch.Tensor, pos: int) -> torch.Tensor:
    """One decode step of emulated ranks: every rank's phase k is issued before
    any rank's phase k+1 (all on the current stream), so a reduce only ever
    waits for pushes launched before it."""
    gens = [m.step_phases(tokens, pos) for m in models]
    live = True
    while live:
        live = False
        for g in gens:
            try:
                next(g)
                live = True
            except StopIteration:
                pass
    return models[0].next_tokens


def shrink(cfg: LlamaConfig, **kw) -> LlamaConfig:
    return replace(cfg, **kw)
