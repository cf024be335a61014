"""Runtime: the quantized GEMV behind the reference's seam.

The reference declares a runtime it never shipped:
``input_sums``, ``qgemv_reference``, ``qgemv(pm, x, sums, threads)`` and
``memory_report``.  This module provides them with the same argument meaning
and errors, backed by libqigen_b200:

* ``qgemv`` accepts any ``PackedMatrix`` (ours or the reference's, either
  ``Layout``).  The first call re-tiles it into the GPU panel layout
   and caches it in ``pm._exec_cache`` — the reference's own hook
  (packing.py:135).  Input sums are fused into the kernel, so ``sums`` is
  accepted for API compatibility and ignored; ``threads`` (CPU column-block
  threads) has no GPU meaning and is only validated.
* numpy in -> numpy out (host round trip, like the reference); CUDA tensor in ->
  CUDA tensor out (stream-ordered, no host sync).
"""

from __future__ import annotations

import operator
import threading
from dataclasses import dataclass

import numpy as np
import torch

from . import _dev
from ._lib import BF16, F16, F32, call, lib
from .config import ConfigError, QuantConfig
from .packing import Layout, PackError, _as_config, _as_words, rowseq_words
from .quant import CodeMatrix, quantize_matrix

_DTYPES = {torch.float32: F32, torch.float16: F16, torch.bfloat16: BF16}
MAX_GEMV_TOKENS = 16
TC_MIN_TOKENS = 16   # north_star (c): tensor cores only from 16 tokens up
MAX_TC_TOKENS = 256


@dataclass
class InputSums:
    """total x-hat and per-group sums."""

    total: float
    per_group: torch.Tensor


def input_sums(x, group_size) -> InputSums:
    """SPEC.md:331-339 on the GPU (fp64 accumulation, one rounding)."""
    xt = _dev.to_device(x, torch.float32)
    if xt.dim() != 1 or xt.numel() == 0:
        raise ConfigError(f"x must be a non-empty vector, got shape {tuple(xt.shape)}")
    n = xt.numel()
    if group_size is not None and n % group_size:
        raise ConfigError(f"group size {group_size} does not divide length {n}")
    G = 1 if group_size is None else n // group_size
    per = torch.empty(G, dtype=torch.float32, device=xt.device)
    tot = torch.empty(1, dtype=torch.float32, device=xt.device)
    st = _dev.stream_handle()
    call("qigen_input_sums", xt.data_ptr(), n, 0 if group_size is None else group_size,
         per.data_ptr(), st)
    call("qigen_input_sums", xt.data_ptr(), n, 0, tot.data_ptr(), st)
    return InputSums(float(tot.item()), per)


class PanelWeights:
    """A weight matrix in the GPU panel layout.

    ``qw``: packed codes, 16-column panels x 256-row supersteps, each lane's
    128-bit words holding whole m16n8k32 A fragments; ``qsz``: (s, z) float2 per
    (panel, group, column).  Built from codes, reference words, or float
    weights (GPU quantize, bit-exact with quant.py)."""

    def __init__(self, qw: torch.Tensor, qsz: torch.Tensor, n: int, m: int, config: QuantConfig):
        self.qw, self.qsz = qw, qsz
        self.n, self.m, self.config = n, m, config

    @property
    def bits(self) -> int:
        return self.config.bits

    @property
    def group_code(self) -> int:
        return self.config.group_code

    @staticmethod
    def _alloc(n, m, config, device):
        L = lib()
        qw = torch.empty(int(L.qigen_panel_words(n, m, config.bits)), dtype=torch.int32, device=device)
        qsz = torch.empty(int(L.qigen_panel_params(n, m, config.group_code)) * 2,
                          dtype=torch.float32, device=device)
        return qw, qsz

    @classmethod
    def from_codes(cls, cm: CodeMatrix) -> "PanelWeights":
        cfg = _as_config(cm.config)
        codes = _dev.to_device(cm.codes, torch.uint8)
        s = _dev.to_device(cm.scales, torch.float32)
        z = _dev.to_device(cm.zeros, torch.float32)
        n, m = codes.shape
        qw, qsz = cls._alloc(n, m, cfg, codes.device)
        call("qigen_panels_from_codes", codes.data_ptr(), s.data_ptr(), z.data_ptr(), n, m,
             cfg.bits, cfg.group_code, qw.data_ptr(), qsz.data_ptr(), _dev.stream_handle())
        return cls(qw, qsz, n, m, cfg)

    @classmethod
    def from_packed(cls, pm) -> "PanelWeights":
        """From a reference-format PackedMatrix (ROW_SEQUENTIAL or ZCURVE words)."""
        cfg = _as_config(pm.config)
        rs = rowseq_words(pm)
        s = _dev.to_device(pm.scales, torch.float32)
        z = _dev.to_device(pm.zeros, torch.float32)
        G = cfg.groups_for_rows(pm.n)
        if tuple(s.shape) != (G, pm.m) or tuple(z.shape) != (G, pm.m):
            raise PackError(f"scales/zeros shape {tuple(s.shape)} != ({G}, {pm.m})")
        qw, qsz = cls._alloc(pm.n, pm.m, cfg, rs.device)
        call("qigen_panels_from_rowseq", rs.data_ptr(), s.data_ptr(), z.data_ptr(), pm.n, pm.m,
             cfg.bits, cfg.group_code, qw.data_ptr(), qsz.data_ptr(), _dev.stream_handle())
        return cls(qw, qsz, pm.n, pm.m, cfg)

    @classmethod
    def from_float(cls, w, config: QuantConfig) -> "PanelWeights":
        """Quantize float weights [n, m] on the GPU and re-tile (no host copy)."""
        cm = quantize_matrix(w, config)
        out = cls.from_codes(cm)
        del cm
        return out

    def to_codes(self) -> torch.Tensor:
        codes = torch.empty((self.n, self.m), dtype=torch.uint8, device=self.qw.device)
        call("qigen_panels_to_codes", self.qw.data_ptr(), self.n, self.m, self.bits,
             codes.data_ptr(), _dev.stream_handle())
        return codes

    def _workspace(self, key, device) -> torch.Tensor:
        """Scratch for prepared activations (owned per matrix and token count,
        so graphs of distinct matrices never share it)."""
        ws = getattr(self, "_ws", None)
        if ws is None:
            ws = self._ws = {}
        buf = ws.get(key)
        if buf is None:
            if isinstance(key, tuple):
                nbytes = int(lib().qigen_gemm_tc_workspace_size(self.n, key[1]))
            else:
                nbytes = int(lib().qigen_gemv_workspace_size(self.n, key))
            buf = ws[key] = torch.empty(nbytes, dtype=torch.uint8, device=device)
        return buf

    def _tc_ok(self) -> bool:
        g = self.config.group_size
        return self.bits == 4 and g in (32, 64, 128, 256)

    def nbytes_algorithmic(self) -> int:
        """Packed codes + f32 scale + f32 zero (the roofline bytes)."""
        G = self.config.groups_for_rows(self.n)
        return self.n * self.m * self.bits // 8 + G * self.m * 8

    def gemv(self, x: torch.Tensor, out: torch.Tensor | None = None, *, accumulate: bool = False,
             k_splits: int = 0, prologue: str | None = None, norm_weight: torch.Tensor | None = None,
             eps: float = 1e-5, x_ready: bool = False, path: str = "auto") -> torch.Tensor:
        """y[t, :] = f(x[t, :]) @ W for t < tokens; x: CUDA [tokens, n] or [n].

        ``path``: ``"auto"`` (tensor-core GEMM from 16 tokens on when the
        config allows it, north_star (c); the exact IMMA GEMV below),
        ``"gemv"`` (always the IMMA GEMV) or ``"tc"`` (always the tensor-core
        GEMM; 4-bit, g in 32..256).

        ``prologue`` fuses the producer-side glue into the GEMV: None (f = id),
        ``"rmsnorm"`` (f = RMSNorm with ``norm_weight``), ``"rmsnorm_folded"``
        (RMSNorm whose weight was folded into W at quantization: y = rsqrt(mean(x^2)
        + eps) (x W), the norm is applied in the epilogue) or ``"swiglu"`` (x holds
        gate | up, [tokens, 2n]; f = silu(gate) * up).  ``x_ready`` asserts that
        x is not the output of the kernel launched just before on this stream
        (independent GEMVs back to back): the GEMV then overlaps that kernel
        completely (QIGEN_GEMV_X_READY)."""
        squeeze = x.dim() == 1
        x2 = x.reshape(1, -1) if squeeze else x
        width = 2 * self.n if prologue == "swiglu" else self.n
        if x2.dim() != 2 or x2.shape[1] != width:
            raise ConfigError(f"x has shape {tuple(x.shape)}, expected [..., {width}]")
        mode = {None: 0, "rmsnorm": 1, "swiglu": 2, "rmsnorm_folded": 3}[prologue]
        if mode == 1 and (norm_weight is None or norm_weight.dtype != torch.float32
                          or not norm_weight.is_cuda or norm_weight.numel() != self.n):
            raise ConfigError("rmsnorm prologue needs a float32 CUDA weight of length n")
        if x2.dtype not in _DTYPES:
            x2 = x2.float()
            x_ready = False  # x is now the conversion kernel's output
        if x2.stride(1) != 1:
            x2 = x2.contiguous()
            x_ready = False
        T = x2.shape[0]
        if out is None:
            out = torch.empty((T, self.m), dtype=torch.float32, device=x2.device)
            accumulate = False
        y2 = out.reshape(T, self.m) if out.dim() == 1 else out
        if y2.dtype != torch.float32 or y2.stride(1) != 1:
            raise ConfigError("out must be float32 with unit column stride")
        if path not in ("auto", "gemv", "tc"):
            raise ConfigError(f"path must be 'auto', 'gemv' or 'tc', got {path!r}")
        if path == "tc" and (mode != 0 or not self._tc_ok()):
            raise ConfigError("the tensor-core path takes 4-bit weights, g in (32, 64, 128, 256) "
                              "and no prologue")
        st = _dev.stream_handle()
        use_tc = path == "tc" or (path == "auto" and T >= TC_MIN_TOKENS and mode == 0
                                  and self._tc_ok())
        if use_tc:
            # small-batch GEMM on the tcgen05 tensor cores (north_star (c))
            for t0 in range(0, T, MAX_TC_TOKENS):
                t1 = min(T, t0 + MAX_TC_TOKENS)
                xs, ys = x2[t0:t1], y2[t0:t1]
                ws = self._workspace(("tc", t1 - t0), x2.device)
                call("qigen_gemm_tc", self.qw.data_ptr(), self.qsz.data_ptr(), self.n, self.m,
                     self.bits, self.group_code, xs.data_ptr(), _DTYPES[xs.dtype], t1 - t0,
                     xs.stride(0), ys.data_ptr(), ys.stride(0), int(accumulate), int(k_splits),
                     ws.data_ptr(), ws.numel(), st)
            return out.reshape(self.m) if squeeze else out
        ws = self._workspace(min(T, MAX_GEMV_TOKENS), x2.device)
        for t0 in range(0, T, MAX_GEMV_TOKENS):
            t1 = min(T, t0 + MAX_GEMV_TOKENS)
            xs, ys = x2[t0:t1], y2[t0:t1]
            call("qigen_gemv_ex", self.qw.data_ptr(), self.qsz.data_ptr(), self.n, self.m,
                 self.bits, self.group_code, xs.data_ptr(), _DTYPES[xs.dtype], t1 - t0,
                 xs.stride(0), ys.data_ptr(), ys.stride(0),
                 int(accumulate) | (X_READY if x_ready else 0), int(k_splits), mode,
                 norm_weight.data_ptr() if mode == 1 else None, float(eps), ws.data_ptr(),
                 ws.numel(), st)
        return out.reshape(self.m) if squeeze else out


    def chain(self, x: torch.Tensor | None, out: torch.Tensor, *, tokens: int,
              accumulate: bool = False, prologue: str | None = None,
              norm_weight: torch.Tensor | None = None, eps: float = 1e-5,
              digits_in: torch.Tensor | None = None, ss_in: torch.Tensor | None = None,
              ss_count: int = 0, digits_out: torch.Tensor | None = None,
              out_scale: torch.Tensor | None = None, out_group: int | None = None,
              ss_out: torch.Tensor | None = None) -> torch.Tensor:
        """One GEMV of a dependent decode chain (qigen_gemv_chain): the consumer
        side reads the activation digits a producer's epilogue wrote
        (``digits_in``, with the producer's sums of squares ``ss_in`` folding an
        RMSNorm into the epilogue); the producer side also writes its final
        output (after the residual add) as the next GEMV's digits
        (``digits_out``, times ``out_scale``) and ``ss_out``."""
        from ._lib import ChainOpts
        import ctypes
        mode = {None: 0, "rmsnorm": 1, "swiglu": 2}[prologue]
        if digits_in is None:
            x2 = x.reshape(tokens, -1)
            xp, xd, ldx = x2.data_ptr(), _DTYPES[x2.dtype], x2.stride(0)
        else:
            xp, xd, ldx = None, F32, self.n
        o = ChainOpts(None if digits_in is None else digits_in.data_ptr(),
                      None if ss_in is None else ss_in.data_ptr(), int(ss_count), float(eps),
                      None if digits_out is None else digits_out.data_ptr(),
                      None if out_scale is None else out_scale.data_ptr(),
                      0 if out_group is None else int(out_group),
                      None if ss_out is None else ss_out.data_ptr())
        ws = self._workspace(min(tokens, MAX_GEMV_TOKENS), out.device)
        y2 = out.reshape(tokens, self.m)
        call("qigen_gemv_chain", self.qw.data_ptr(), self.qsz.data_ptr(), self.n, self.m,
             self.bits, self.group_code, xp, xd, tokens, ldx, y2.data_ptr(), y2.stride(0),
             int(accumulate), mode, norm_weight.data_ptr() if mode == 1 else None, float(eps),
             ws.data_ptr(), ws.numel(), ctypes.byref(o), _dev.stream_handle())
        return out

    def push(self, comm, slot: int, x: torch.Tensor, *, prologue: str | None = None,
             norm_weight: torch.Tensor | None = None, eps: float = 1e-5) -> None:
        """Row-parallel partial x W of a tensor-parallel rank, stored by the GEMV
        epilogue into slot `slot` of every rank's inbox (qigen_gemv_tp_push;
        the reduce is ``comm.reduce``).  x: CUDA [tokens, n] (or [tokens, 2n]
        for the SwiGLU prologue)."""
        x2 = x.reshape(1, -1) if x.dim() == 1 else x
        width = 2 * self.n if prologue == "swiglu" else self.n
        if x2.dim() != 2 or x2.shape[1] != width or x2.dtype not in _DTYPES or x2.stride(1) != 1:
            raise ConfigError(f"x must be a unit-stride CUDA [tokens, {width}] f32/f16/bf16 tensor")
        mode = {None: 0, "rmsnorm": 1, "swiglu": 2}[prologue]
        T = x2.shape[0]
        ws = self._workspace(min(T, MAX_GEMV_TOKENS), x2.device)
        call("qigen_gemv_tp_push", comm._h, int(slot), self.qw.data_ptr(), self.qsz.data_ptr(),
             self.n, self.m, self.bits, self.group_code, x2.data_ptr(), _DTYPES[x2.dtype], T,
             x2.stride(0), mode, norm_weight.data_ptr() if mode == 1 else None, float(eps),
             ws.data_ptr(), ws.numel(), _dev.stream_handle())


X_READY = 2  # QIGEN_GEMV_X_READY (include/qigen_b200.h)


def digits_buffer(n: int, tokens: int, device) -> torch.Tensor:
    """Zero-filled prepared-digit buffer for a GEMV with K = n (qigen_gemv_chain)."""
    return torch.zeros(int(lib().qigen_gemv_workspace_size(n, tokens)), dtype=torch.uint8,
                       device=device)


def ss_count(m: int) -> int:
    """Per-CTA sums of squares a chain producer with m outputs writes per token."""
    return int(lib().qigen_gemv_ss_count(m))


class GemvGroup:
    """Independent GEMVs y_i = x_i @ W_i run as ONE persistent launch
    (qigen_gemv_group_*): the replacement for a loop of independent
    ``qgemv(pm_i, x_i)`` calls.  ``entries`` are
    ``(PanelWeights, x, y)`` with x CUDA [n] / [tokens <= 2, n] and y f32
    [m] / [tokens, m]; the tensors are referenced, not copied, so later writes
    to x are seen by the next ``run()``.  ``run()`` is stream-ordered and
    graph-capturable."""

    def __init__(self, entries, *, pinned_x: bool = False):
        import ctypes

        from ._lib import GemvDesc
        self._keep = []
        descs = (GemvDesc * len(entries))()
        for i, (pw, x, y) in enumerate(entries):
            x2 = x.reshape(1, -1) if x.dim() == 1 else x
            y2 = y.reshape(1, -1) if y.dim() == 1 else y
            x_ok = x2.is_cuda or (pinned_x and x2.is_pinned())  # pinned: read over PCIe
            if x2.dtype not in _DTYPES or x2.stride(1) != 1 or not x_ok:
                raise ConfigError("group x must be a CUDA f32/f16/bf16 tensor with unit stride")
            y_ok = y2.is_cuda or y2.is_pinned()  # pinned: stored over PCIe (zero-copy)
            if y2.dtype != torch.float32 or y2.stride(1) != 1 or y2.shape != (x2.shape[0], pw.m):
                raise ConfigError(f"group y must be float32 [{x2.shape[0]}, {pw.m}]")
            if not y_ok:
                raise ConfigError("group y must be a CUDA tensor or pinned host memory")
            if x2.shape[1] != pw.n:
                raise ConfigError(f"x has {x2.shape[1]} columns, expected {pw.n}")
            descs[i] = GemvDesc(pw.qw.data_ptr(), pw.qsz.data_ptr(), pw.n, pw.m, pw.bits,
                                pw.group_code, x2.data_ptr(), _DTYPES[x2.dtype], x2.shape[0],
                                x2.stride(0), y2.data_ptr(), y2.stride(0))
            self._keep += [pw, x, y]
        h = ctypes.c_void_p()
        call("qigen_gemv_group_create", len(entries), ctypes.addressof(descs), ctypes.byref(h))
        self._h = h
        self.nbytes_algorithmic = sum(pw.nbytes_algorithmic() for pw, _, _ in entries)

    @staticmethod
    def supports(pw: "PanelWeights") -> bool:
        """The grouped kernel's configurations: every group size the GEMV takes
        except g = 16 (whose per-half-step flush the grouped records do not carry)."""
        return pw.config.group_size != 16

    def run(self) -> None:
        call("qigen_gemv_group_run", self._h, _dev.stream_handle())

    def __del__(self):
        h = getattr(self, "_h", None)
        if h:
            try:
                lib().qigen_gemv_group_destroy(h)
            except Exception:  # noqa: BLE001
                pass


def exec_layout(pm) -> PanelWeights:
    """The cached GPU layout of a PackedMatrix (packing.py:135 hook)."""
    cache = getattr(pm, "_exec_cache", None)
    if isinstance(cache, PanelWeights) and cache.qw.device.index == torch.cuda.current_device():
        return cache
    pw = PanelWeights.from_packed(pm)
    try:
        pm._exec_cache = pw
    except AttributeError:
        pass
    return pw


def qgemv(pm, x, sums=None, threads=None, *, out=None, accumulate: bool = False):
    """y = x W through the GPU kernel.

    ``x``: [n] or [tokens, n] (numpy, or CUDA tensor in f32/f16/bf16).
    Returns numpy for host input, a CUDA f32 tensor for device input.
    """
    if threads is not None and (not isinstance(threads, (int, np.integer)) or threads < 1):
        raise ConfigError(f"thread count must be >= 1, got {threads!r}")
    host = _dev.is_host(x)
    if isinstance(x, torch.Tensor) and host:
        # CPU torch tensor (possibly pinned): async H2D, result returned as a CPU tensor
        if x.shape[-1] != pm.n or x.dim() not in (1, 2):
            raise ConfigError(f"x has shape {tuple(x.shape)}, expected [..., {pm.n}]")
        xt = x.to(device=_dev.require_cuda(), dtype=torch.float32, non_blocking=True)
        y = exec_layout(pm).gemv(xt)
        if out is not None:
            out.copy_(y)
            return out
        return y.cpu()
    if host:
        xa = np.asarray(x, dtype=np.float32)
        if xa.ndim not in (1, 2) or xa.shape[-1] != pm.n:
            raise ConfigError(f"x has shape {xa.shape}, expected [{pm.n}] or [tokens, {pm.n}]")
        if not np.all(np.isfinite(xa)):
            raise ConfigError("x contains non-finite values")
        if xa.ndim == 1 and out is None and not accumulate:
            # one host vector: the zero-copy path of qgemv_batch with a plan kept per
            # matrix (x gathered into pinned memory that the kernel reads over PCIe, y
            # stored into a fresh pinned block; no staged H2D / D2H copies)
            pw = exec_layout(pm)
            if GemvGroup.supports(pw):
                b = getattr(pw, "_single", None)
                if b is None:
                    b = pw._single = _Batch([pm], _dev.require_cuda())
                with b.lock:
                    return _batch_call(b, [xa])[0]
        xt = _dev.to_device(xa, torch.float32)
    else:
        xt = x
        if xt.shape[-1] != pm.n or xt.dim() not in (1, 2):
            raise ConfigError(f"x has shape {tuple(xt.shape)}, expected [..., {pm.n}]")
    pw = exec_layout(pm)
    squeeze = xt.dim() == 1
    x2 = xt.reshape(1, -1) if squeeze else xt
    y = pw.gemv(x2, out=None if host or out is None else out.reshape(x2.shape[0], pm.m),
                accumulate=accumulate and out is not None)
    if squeeze:
        y = y.reshape(pm.m)
    if host:
        yh = _dev.to_host(y)
        if out is not None:
            np.copyto(out, yh)
            return out
        return yh
    return y


class _Batch:
    """Device staging + grouped plan for one list of PackedMatrix objects."""

    def __init__(self, pms, dev):
        self.pms = list(pms)  # keeps the objects (and their ids) alive
        self.pws = [exec_layout(pm) for pm in self.pms]
        self.koff = np.cumsum([0] + [pw.n for pw in self.pws])
        self.noff = np.cumsum([0] + [pw.m for pw in self.pws])
        # per-matrix slices of the result block (np.split costs ~1 us per piece)
        self.xshapes = [(pw.n,) for pw in self.pws]
        self.xtypes = [np.ndarray] * len(self.pws)
        self.yslices = [slice(int(a), int(e)) for a, e in zip(self.noff[:-1], self.noff[1:])]
        self.x = torch.zeros(int(self.koff[-1]), device=dev)
        self.y = torch.zeros(int(self.noff[-1]), device=dev)
        self.xh = torch.zeros(int(self.koff[-1])).pin_memory()
        self.xh_np = self.xh.numpy()
        self._group = self._group_host = None
        # the staging buffers, the plans' activation records and schedule
        # counter are per list: concurrent calls on one list take turns
        self.lock = threading.Lock()
        self.done = None  # event after the last device-path call (other streams wait on it)
        # matrices the grouped kernel takes, and the rest (g = 16: a flush every
        # half step; run as single GEMVs right after the grouped launch)
        self.gi = [i for i, pw in enumerate(self.pws) if GemvGroup.supports(pw)]
        self.si = [i for i in range(len(self.pws)) if i not in set(self.gi)]

    def _xs(self, buf, i):
        return buf[self.koff[i]:self.koff[i + 1]]

    def _ys(self, buf, i):
        return buf[self.noff[i]:self.noff[i + 1]]

    @property
    def group(self) -> "GemvGroup | None":
        """Grouped launch over device inputs (``x``), built on first use."""
        if self._group is None and self.gi:
            self._group = GemvGroup([(self.pws[i], self._xs(self.x, i), self._ys(self.y, i))
                                     for i in self.gi])
        return self._group

    def run_device(self) -> None:
        if self.group is not None:
            self.group.run()
        for i in self.si:
            self.pws[i].gemv(self._xs(self.x, i), out=self._ys(self.y, i))

    @property
    def group_host(self) -> "GemvGroup":
        """Grouped launch whose prep kernel reads the pinned gather buffer
        (``xh``) over PCIe: no H2D copy (tools/zc_exp.py: 218 vs 236-240 us per
        call on the configs[1] sweep, identical outputs)."""
        if self._group_host is None:
            # outputs: a pinned template block; each call rebases the plan's y
            # onto a fresh pinned block (qigen_gemv_group_run_rebased)
            self.yh0 = torch.empty(self.y.numel(), pin_memory=True)
            self.yh0_ptr = self.yh0.data_ptr()
            self._group_host = GemvGroup([(self.pws[i], self._xs(self.xh, i),
                                           self._ys(self.yh0, i)) for i in self.gi],
                                         pinned_x=True) if self.gi else None
        return self._group_host


def _batch_host_run(b: "_Batch"):
    """The grouped launch reading the gathered inputs from pinned host memory
    and writing the results into a fresh pinned block (zero-copy both ways)."""
    gh = b.group_host
    # results land in a fresh pinned block (torch's caching host allocator:
    # no cudaHostAlloc after warm-up) that the returned views own, so no
    # host-side copy out of a shared staging buffer is needed.
    yh = torch.empty(b.y.numel(), pin_memory=True)
    if gh is not None:
        call("qigen_gemv_group_run_rebased", gh._h, b.yh0_ptr, yh.data_ptr(),
             _dev.stream_handle())
    for i in b.si:  # matrices outside the grouped kernel: single GEMVs, staged copies
        xd = b._xs(b.x, i)
        xd.copy_(b._xs(b.xh, i), non_blocking=True)
        b._ys(yh, i).copy_(b.pws[i].gemv(xd), non_blocking=True)
    torch.cuda.current_stream().synchronize()
    yv = yh.numpy()
    return [yv[s] for s in b.yslices]


_BATCHES: dict = {}
_MAX_BATCHES = 8
_LAST = [None, None]  # (matrix list object, _Batch) of the previous call
_SHAPE = operator.attrgetter("shape")


class PinnedInputs(list):
    """The activation vectors of one matrix list as numpy views of its page-locked
    gather buffer (``qgemv_batch_inputs``)."""

    _batch = None


def qgemv_batch_inputs(pms) -> "PinnedInputs":
    """Page-locked input vectors for ``qgemv_batch(pms, .)``: a list of numpy [n_i]
    views of the matrix list's pinned gather buffer.  Fill them in place (they are
    ordinary numpy arrays) and pass the list itself to ``qgemv_batch``: the grouped
    launch then reads them over PCIe directly, with no host-side gather.  The
    buffer belongs to the matrix list: one caller at a time."""
    if not pms:
        raise ConfigError("qgemv_batch needs one activation vector per matrix")
    with _CACHE_LOCK:
        b = _lookup_batch(pms)
    xs = PinnedInputs(b.xh_np[int(a):int(e)] for a, e in zip(b.koff[:-1], b.koff[1:]))
    xs._batch = b
    return xs


def qgemv_batch(pms, xs):
    """Independent ``qgemv(pm_i, x_i)`` calls for a list of
    matrices, as ONE grouped GPU launch (``GemvGroup``).  ``xs``: per matrix an
    [n_i] activation vector (numpy / CPU tensor, or CUDA f32 tensor).  Host
    inputs are gathered into one pinned buffer that the grouped launch reads
    over PCIe, and the kernel stores y straight into a fresh pinned block
    (zero-copy both ways: no H2D or D2H copy); the numpy results are views of
    that block, so they stay valid across later calls.  Device inputs give
    CUDA tensors.  The grouped plan and staging buffers are cached per matrix
    list (the 8 most recently used lists); concurrent calls from several
    threads are safe (calls on the same list are serialised).  Inputs obtained
    from ``qgemv_batch_inputs(pms)`` (numpy views of the pinned buffer, filled in
    place) skip the gather."""
    if len(pms) != len(xs) or not pms:
        raise ConfigError("qgemv_batch needs one activation vector per matrix")
    with _CACHE_LOCK:
        b = _lookup_batch(pms)
    with b.lock:
        if type(xs) is PinnedInputs and xs._batch is b:
            return _batch_host_run(b)  # the inputs already are the pinned buffer
        return _batch_call(b, xs)


_CACHE_LOCK = threading.Lock()


def _lookup_batch(pms) -> "_Batch":
    b = _LAST[1]
    # same matrix list as the previous call: it is already the most recently used
    if not (_LAST[0] is pms and len(pms) == len(b.pms) and all(map(operator.is_, pms, b.pms))):
        key = tuple(map(id, pms))
        b = _BATCHES.pop(key, None)
        if b is None or any(p is not q for p, q in zip(b.pms, pms)):
            b = _Batch(pms, _dev.require_cuda())  # fails loudly without a GPU
        _BATCHES[key] = b  # most recently used last
        while len(_BATCHES) > _MAX_BATCHES:  # bounded: plans pin their matrices and buffers
            _BATCHES.pop(next(iter(_BATCHES)))
        _LAST[0], _LAST[1] = pms, b
    return b


def _batch_call(b: "_Batch", xs):
    if len(xs) != len(b.pws):
        raise ConfigError("qgemv_batch needs one activation vector per matrix")
    if list(map(type, xs)) == b.xtypes and list(map(_SHAPE, xs)) == b.xshapes:
        # fast path: every x a host numpy vector of the right length
        np.concatenate(xs, out=b.xh_np, casting="same_kind")
        return _batch_host_run(b)
    host = True
    hx = []  # host arrays for the gather
    for i, (pw, x) in enumerate(zip(b.pws, xs)):
        if type(x) is not np.ndarray:
            if isinstance(x, torch.Tensor):
                if x.is_cuda:
                    host = False
                else:
                    x = x.numpy()
            else:
                x = np.asarray(x)
        if x.shape != (pw.n,):
            raise ConfigError(f"x[{i}] has shape {tuple(x.shape)}, expected [{pw.n}]")
        hx.append(x)
    if host:
        # one host-side gather into the pinned staging buffer, then the
        # zero-copy grouped launch
        np.concatenate(hx, out=b.xh_np, casting="same_kind")
        return _batch_host_run(b)
    # device path: stream-ordered, no host sync; a call on another stream
    # first waits for the previous call's use of the shared buffers
    cur = torch.cuda.current_stream()
    if b.done is not None:
        cur.wait_event(b.done)
    torch.cat([x.reshape(-1).float() for x in xs], out=b.x)
    b.run_device()
    out = list(torch.split(b.y.clone(), [pw.m for pw in b.pws]))
    b.done = torch.cuda.Event()
    b.done.record(cur)
    return out


def qgemv_reference(pm, x):
    """the unfactored dense oracle, on the GPU — full
    dequantization (quant.py:130-138) then an fp64 matrix product."""
    from .packing import extract_codes
    from .quant import dequantize_matrix
    host = _dev.is_host(x)
    xt = _dev.to_device(x, torch.float64)
    if xt.shape[-1] != pm.n:
        raise ConfigError(f"dimension mismatch: x has {xt.shape[-1]} entries, W has {pm.n} rows")
    wd = dequantize_matrix(extract_codes(pm)).double()
    y = xt @ wd
    return _dev.to_host(y) if host else y


def memory_report(pm) -> dict:
    """payload decomposition and compression vs. 32 n m."""
    wb, sb, zb = pm.payload_bits()
    total = wb + sb + zb
    return {"weight_bits": wb, "scale_bits": sb, "zero_bits": zb, "total_bits": total,
            "fp32_bits": 32 * pm.n * pm.m, "ratio": 32 * pm.n * pm.m / total}
