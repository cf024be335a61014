"""CPU oracle for the QIGen hot path — TEST INFRASTRUCTURE ONLY.

This module restates, in plain numpy, the reference algorithms that sit on the
quantized-GEMV path of QIGen (arXiv 2307.03738, reference at
``/root/reference/pkg/src/qigen``).  Only ``tests/``, ``__graft_entry__.smoke()``
and the ``cpu_baseline`` / ``--impl reference`` legs of ``bench.py`` may import
it, and only as the *checker*.  The product package
(``paper_2307_03738_b200``) never imports anything from ``oracle/``.

Parity pin: every integer function here (quantize, pack, permute, plan) is
checked bit-for-bit against fixtures produced by running the reference itself
(``tests/golden/make_golden.py``, committed together with the ``.npz`` files it
wrote).  The floating-point qGEMV port in ``qgemv_port.c`` is checked bit-for-bit
against the reference's generated kernel run on the same inputs (same fixtures).

Each function names the reference ``file:line`` it restates.
"""

from __future__ import annotations

import ctypes
import math
import os
from pathlib import Path

import numpy as np

HERE = Path(__file__).resolve().parent

SUPPORTED_BITS = (2, 3, 4)
REAL32, QUANTIZED = "real32", "quantized"


# ---------------------------------------------------------------------------
# config.py
# ---------------------------------------------------------------------------

def pack_unit(bits: int) -> tuple[int, int]:
    """(codes, words) per packing unit — config.py:91-100."""
    if bits == 3:
        return 32, 3
    if bits in (2, 4):
        return 32 // bits, 1
    raise ValueError(bits)


def groups_for_rows(n: int, group_size) -> int:
    """config.py:68-75 (None = FULL_COLUMN, one group per column)."""
    if group_size is None:
        return 1
    if n % group_size:
        raise ValueError(f"group size {group_size} does not divide {n}")
    return n // group_size


# ---------------------------------------------------------------------------
# quant.py
# ---------------------------------------------------------------------------

def round_half_away(v: np.ndarray) -> np.ndarray:
    """quant.py:70-71: copysign(floor(|v| + 0.5), v) in float64."""
    return np.copysign(np.floor(np.abs(v) + 0.5), v)


def clip_keep_sign(v: np.ndarray, lo: float, hi: float) -> np.ndarray:
    """np.clip semantics used at quant.py:87,91 — a value equal to a bound
    (e.g. -0.0 vs 0.0) is returned unchanged, so signed zeros survive."""
    out = np.where(v < lo, lo, v)
    return np.where(out > hi, hi, out)


def quantize_blocks(x: np.ndarray, bits: int, zero_mode: str):
    """quant.py:74-94, groups along axis 1 of a (groups, g, m) float32 array.

    fp64 min/max; s = 1 for a constant group else span/max_code (fp64);
    narrowed to fp32; z = -min / f64(s32); REAL32 keeps f32(z), QUANTIZED
    rounds half-away and clips to [0, max_code]; codes = clip(rha(x/s32+z32)).
    """
    max_code = (1 << bits) - 1
    x64 = x.astype(np.float64)
    mn = x64.min(axis=1, keepdims=True)
    mx = x64.max(axis=1, keepdims=True)
    span = mx - mn
    s = np.where(span == 0.0, 1.0, span / max_code)
    s32 = s.astype(np.float32)
    z = -mn / s32.astype(np.float64)
    if zero_mode == QUANTIZED:
        z32 = clip_keep_sign(round_half_away(z), 0.0, float(max_code)).astype(np.float32)
    else:
        z32 = z.astype(np.float32)
    v = x64 / s32.astype(np.float64) + z32.astype(np.float64)
    codes = clip_keep_sign(round_half_away(v), 0.0, float(max_code)).astype(np.uint8)
    return codes, s32[:, 0, :], z32[:, 0, :]


def quantize_matrix(w: np.ndarray, bits: int, group_size, zero_mode: str = REAL32):
    """quant.py:119-127 — returns (codes[n,m] u8, scales[G,m] f32, zeros[G,m] f32)."""
    w = np.asarray(w, dtype=np.float32)
    n, m = w.shape
    G = groups_for_rows(n, group_size)
    codes, s, z = quantize_blocks(w.reshape(G, n // G, m), bits, zero_mode)
    return codes.reshape(n, m), s, z


def dequantize_matrix(codes, scales, zeros) -> np.ndarray:
    """quant.py:130-138: f32(s * (f32(c) - z)) per group."""
    n, m = codes.shape
    G = scales.shape[0]
    c = codes.reshape(G, n // G, m).astype(np.float32)
    out = scales[:, None, :] * (c - zeros[:, None, :])
    return out.reshape(n, m).astype(np.float32)


# ---------------------------------------------------------------------------
# packing.py
# ---------------------------------------------------------------------------

def pack_words(codes: np.ndarray, bits: int) -> np.ndarray:
    """packing.py:42-70.  2/4-bit: code j of a word at bits [j*b, (j+1)*b).
    3-bit: 32 codes form a little-endian 96-bit stream (bit 3j+t = bit t of
    code j) split into three words.  Restated with explicit bit arithmetic."""
    c = np.asarray(codes, dtype=np.uint64).reshape(-1)
    unit, kw = pack_unit(bits)
    if c.size % unit:
        raise ValueError("code count not a multiple of the packing unit")
    if bits != 3:
        c = c.reshape(-1, unit)
        sh = (np.arange(unit, dtype=np.uint64) * np.uint64(bits))
        return (c << sh).sum(axis=1).astype(np.uint32)
    c = c.reshape(-1, 32)
    out = np.zeros((c.shape[0], 3), dtype=np.uint64)
    for j in range(32):
        bit = 3 * j
        k, off = divmod(bit, 32)
        out[:, k] |= (c[:, j] << np.uint64(off)) & np.uint64(0xFFFFFFFF)
        if off > 29:  # straddles into the next word
            out[:, k + 1] |= c[:, j] >> np.uint64(32 - off)
    return out.astype(np.uint32).reshape(-1)


def unpack_words(words: np.ndarray, bits: int) -> np.ndarray:
    """packing.py:73-90, exact inverse of pack_words (straddle rule as in
    kernelgen.py:116-124)."""
    w = np.asarray(words, dtype=np.uint64).reshape(-1)
    unit, kw = pack_unit(bits)
    mask = np.uint64((1 << bits) - 1)
    if bits != 3:
        sh = np.arange(unit, dtype=np.uint64) * np.uint64(bits)
        return ((w[:, None] >> sh) & mask).astype(np.uint8).reshape(-1)
    w = w.reshape(-1, 3)
    out = np.empty((w.shape[0], 32), dtype=np.uint8)
    for j in range(32):
        bit = 3 * j
        k, off = divmod(bit, 32)
        v = w[:, k] >> np.uint64(off)
        if off > 29:
            lo = 32 - off
            v = v | ((w[:, k + 1] & np.uint64((1 << (3 - lo)) - 1)) << np.uint64(lo))
        out[:, j] = (v & mask).astype(np.uint8)
    return out.reshape(-1)


def pack_rowseq(codes: np.ndarray, bits: int) -> np.ndarray:
    """packing.py:204-214: ROW_SEQUENTIAL words, word (r, k, c) at
    (r*Kw + k)*m + c — a [K*b/32, N] uint32 matrix, K-packing inside a word."""
    n, m = codes.shape
    unit, kw = pack_unit(bits)
    if n % unit:
        raise ValueError("row count must fill whole packing units")
    per_col = pack_words(np.ascontiguousarray(codes.T).reshape(-1), bits)
    return np.ascontiguousarray(per_col.reshape(m, -1).T).reshape(-1)


def unpack_rowseq(words: np.ndarray, n: int, m: int, bits: int) -> np.ndarray:
    """Inverse of pack_rowseq (packing.py:236-240)."""
    by_col = np.ascontiguousarray(np.asarray(words).reshape(-1, m).T).reshape(-1)
    return np.ascontiguousarray(unpack_words(by_col, bits).reshape(m, n).T)


def _spread(v: int) -> int:
    out = 0
    for i in range(32):
        out |= ((v >> i) & 1) << (2 * i)
    return out


def morton_index(rb: int, cb: int) -> int:
    """packing.py:93-107: row bits -> even positions, column bits -> odd."""
    return _spread(rb) | (_spread(cb) << 1)


def block_order(rbs: int, cbs: int) -> list[tuple[int, int]]:
    """packing.py:110-114."""
    return sorted(((r, c) for r in range(rbs) for c in range(cbs)),
                  key=lambda rc: morton_index(*rc))


def grid(n: int, m: int, m_b: int, t_b: int) -> tuple[int, int]:
    """packing.py:159-160."""
    return -(-n // m_b), -(-m // t_b)


def storage_permutation(n, m, bits, m_b, t_b, zcurve: bool) -> np.ndarray:
    """packing.py:175-201: storage position -> ROW_SEQUENTIAL position.
    ZCURVE stores Morton-ordered blocks compactly (ragged edges not padded),
    each block as [word-row][k][col]."""
    unit, kw = pack_unit(bits)
    wr = n // unit
    if not zcurve:
        return np.arange(wr * kw * m, dtype=np.int64)
    wgb = m_b // unit
    rbs, cbs = grid(n, m, m_b, t_b)
    parts = []
    for rb, cb in block_order(rbs, cbs):
        r = np.arange(rb * wgb, min((rb + 1) * wgb, wr), dtype=np.int64)
        c = np.arange(cb * t_b, min((cb + 1) * t_b, m), dtype=np.int64)
        k = np.arange(kw, dtype=np.int64)
        parts.append(((r[:, None, None] * kw + k[None, :, None]) * m
                      + c[None, None, :]).reshape(-1))
    return np.concatenate(parts)


def lay_out_words(codes: np.ndarray, bits: int, m_b: int, t_b: int, zcurve: bool):
    """packing.py:217-226 (words only)."""
    n, m = codes.shape
    rowseq = pack_rowseq(codes, bits)
    return rowseq[storage_permutation(n, m, bits, m_b, t_b, zcurve)]


def words_to_rowseq(words, n, m, bits, m_b, t_b, zcurve: bool) -> np.ndarray:
    """Inverse permutation, packing.py:233-235."""
    perm = storage_permutation(n, m, bits, m_b, t_b, zcurve)
    out = np.empty_like(np.asarray(words))
    out[perm] = words
    return out


# ---------------------------------------------------------------------------
# perfmodel.py (the plan fixes the reference ZCURVE layout)
# ---------------------------------------------------------------------------

def plan(bits: int, group_size, dims, l1_bits=262144, vregs=16, lanes=8):
    """perfmodel.py:128-214 with the default HardwareSpec (:33-36).
    Register tile: maximise m_u*t_u (then t_u) s.t. m_u + m_u*t_u + t_u <= vregs.
    Cache block: maximise 32 m_b + b m_b t_b + 32 t_b <= l1_bits over multiples
    of the aligned steps, capped at the dims; ties -> larger t_b, larger m_b."""
    best_rt = None
    for mu in range(1, vregs + 1):
        for tu in range(1, vregs + 1):
            if mu + mu * tu + tu <= vregs:
                key = (mu * tu, tu)
                if best_rt is None or key > best_rt[0]:
                    best_rt = (key, (mu, tu))
    mu, tu = best_rt[1]
    unit, _ = pack_unit(bits)
    m_align = unit if group_size is None else math.lcm(unit, group_size)
    m_step = math.lcm(mu, m_align)
    t_step = math.lcm(tu, tu * lanes)
    n, m = dims
    m_cap = max(m_step, (n // m_step) * m_step)
    t_cap = max(t_step, (m // t_step) * t_step)
    best = None
    for m_b in range(m_step, m_cap + 1, m_step):
        t_fit = (l1_bits - 32 * m_b) // (bits * m_b + 32) if l1_bits > 32 * m_b else 0
        t_b = min(t_cap, (t_fit // t_step) * t_step)
        if t_b < t_step:
            continue
        key = (32 * m_b + bits * m_b * t_b + 32 * t_b, t_b, m_b)
        if best is None or key > best:
            best = key
    if best is None:
        raise ValueError("no feasible cache block")
    return mu, tu, best[2], best[1]


# ---------------------------------------------------------------------------
# runtime (missing in the reference)
# ---------------------------------------------------------------------------

def input_sums(x: np.ndarray, group_size) -> np.ndarray:
    """per-group sums of x (FULL_COLUMN: the total x-hat).
    Accumulated in fp64 and rounded once to fp32."""
    x = np.asarray(x, dtype=np.float32)
    if group_size is None:
        return np.array([x.astype(np.float64).sum()], dtype=np.float32)
    return x.astype(np.float64).reshape(-1, group_size).sum(axis=1).astype(np.float32)


def qgemv_reference(codes, scales, zeros, x) -> np.ndarray:
    """unfactored dense oracle y = x @ dequantize(W), fp64."""
    wd = dequantize_matrix(codes, scales, zeros).astype(np.float64)
    return np.asarray(x, dtype=np.float64) @ wd


class ExecLayout:
    """the padded execution layout the reference's generated
    kernel reads (full m_b x t_b blocks in Morton order, ghost codes 0, ghost
    scales 1 / zeros 0) plus its block descriptors (kernelgen.py:399-413)."""

    def __init__(self, rowseq_words, scales, zeros, n, m, bits, group_size, m_b, t_b):
        unit, kw = pack_unit(bits)
        self.n, self.m, self.bits, self.g = n, m, bits, group_size
        self.m_b, self.t_b = m_b, t_b
        rbs, cbs = grid(n, m, m_b, t_b)
        self.rbs, self.cbs = rbs, cbs
        self.n_pad, self.m_pad = rbs * m_b, cbs * t_b
        wgb = m_b // unit
        bw = wgb * kw * t_b
        rs = np.asarray(rowseq_words, dtype=np.uint32).reshape(n // unit, kw, m)
        full = np.zeros((self.n_pad // unit, kw, self.m_pad), dtype=np.uint32)
        full[: n // unit, :, :m] = rs
        order = block_order(rbs, cbs)
        words = np.empty(len(order) * bw, dtype=np.uint32)
        for bi, (rb, cb) in enumerate(order):
            words[bi * bw:(bi + 1) * bw] = full[rb * wgb:(rb + 1) * wgb, :,
                                                cb * t_b:(cb + 1) * t_b].reshape(-1)
        self.words = words
        self.blk_off = np.arange(len(order), dtype=np.int64) * bw
        self.blk_rb = np.array([rb for rb, _ in order], dtype=np.int64)
        self.blk_cb = np.array([cb for _, cb in order], dtype=np.int64)
        G = scales.shape[0]
        g_pad = 1 if group_size is None else self.n_pad // group_size
        self.scales = np.ones((g_pad, self.m_pad), dtype=np.float32)
        self.zeros = np.zeros((g_pad, self.m_pad), dtype=np.float32)
        self.scales[:G, :m] = scales
        self.zeros[:G, :m] = zeros

    def pad_x(self, x):
        xp = np.zeros(self.n_pad, dtype=np.float32)
        xp[: self.n] = x
        return xp

    def xsums(self, x_pad):
        return input_sums(x_pad, self.g)


# ---------------------------------------------------------------------------
# C port of the generated kernel (qgemv_port.c)
# ---------------------------------------------------------------------------

_LIB = None


def _lib():
    global _LIB
    if _LIB is None:
        path = HERE / "libqgemv_port.so"
        if not path.exists():
            build_port()
        _LIB = ctypes.CDLL(str(path))
        p = ctypes.c_void_p
        i64 = ctypes.c_int64
        i32 = ctypes.c_int
        _LIB.qgemv_port_blocks.argtypes = [p, p, p, p, p, p, i32, i32, i32, i32, i32,
                                           p, p, p, i64, i64, i64, i64]
        _LIB.qgemv_port_blocks.restype = None
        _LIB.qgemv_port_threads.argtypes = [p, p, p, p, p, p, i32, i32, i32, i32, i32,
                                            p, p, p, i64, i64, i32]
        _LIB.qgemv_port_threads.restype = None
        _LIB.qgemv_port_max_threads.restype = i32
    return _LIB


def build_port() -> Path:
    """Compile qgemv_port.c with gcc (no FMA contraction: the reference kernel
    rounds the product and the sum separately)."""
    src = HERE / "qgemv_port.c"
    out = HERE / "libqgemv_port.so"
    cmd = (f"gcc -O3 -march=native -ffp-contract=off -fno-fast-math -fopenmp -shared -fPIC "
           f"-o {out} {src}")
    if os.system(cmd) != 0:
        raise RuntimeError(f"oracle build failed: {cmd}")
    return out


def port_max_threads() -> int:
    return int(_lib().qgemv_port_max_threads())


def qgemv_port(ex: ExecLayout, x: np.ndarray, threads: int = 1, xsums=None) -> np.ndarray:
    """Run the C port of the reference's generated kernel (grouped:
    kernelgen.py:264-313 + flush :227-240; FC: :243-261 with the x-index fix
    of SURVEY F4 + epilogue :316-330) over the exec layout.  Column blocks are
    split into `threads` contiguous ranges like the reference runtime
    (SPEC.md:376).  Returns y[:m] (float32)."""
    xp = ex.pad_x(x)
    xs = ex.xsums(xp) if xsums is None else np.asarray(xsums, dtype=np.float32)
    y = np.zeros(ex.m_pad, dtype=np.float32)
    mu, tu = 3, 3
    lib = _lib()
    g = 0 if ex.g is None else ex.g
    lib.qgemv_port_threads(ex.words.ctypes.data, ex.scales.ctypes.data, ex.zeros.ctypes.data,
                           xp.ctypes.data, xs.ctypes.data, y.ctypes.data,
                           ex.bits, g, ex.m_b, ex.t_b, tu * 8,
                           ex.blk_off.ctypes.data, ex.blk_rb.ctypes.data, ex.blk_cb.ctypes.data,
                           len(ex.blk_off), ex.cbs, int(threads))
    return y[: ex.m].copy()
