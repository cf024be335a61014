"""Bit-packing and blocked layouts on the GPU, bit-exact with the reference
(``qigen/packing.py``): ROW_SEQUENTIAL words = GPTQ-style [K*b/32, N] uint32
matrix, ZCURVE = Morton-ordered m_b x t_b blocks stored compactly.

``PackedMatrix`` keeps the reference's fields (packing.py:117-156); its
``_exec_cache`` (packing.py:135) holds the GPU panel layout built on the first
``qgemv``.
"""

from __future__ import annotations

import enum
from dataclasses import dataclass, field

import numpy as np
import torch

from . import _dev
from ._lib import call
from .config import ConfigError, QuantConfig, check_row_count, pack_unit
from .perfmodel import TilePlan
from .quant import CodeMatrix


class Layout(enum.Enum):
    ROW_SEQUENTIAL = 0
    ZCURVE = 1


class PackError(ValueError):
    """Packing input violates a layout precondition (packing.py:35)."""


def _check_bits(bits: int) -> None:
    if bits not in (2, 3, 4):
        raise ConfigError(f"unsupported bit width {bits}")


def pack_words(codes, bits: int) -> torch.Tensor:
    """packing.py:42-70 (one column of the row-sequential packer)."""
    _check_bits(bits)
    c = _dev.to_device(codes, torch.int64)
    if c.dim() != 1:
        raise PackError(f"codes must be 1-D, got shape {tuple(c.shape)}")
    unit, _ = pack_unit(bits)
    if c.numel() % unit:
        raise PackError(f"code count {c.numel()} is not a multiple of {unit}")
    if c.numel() == 0:
        return torch.empty(0, dtype=torch.int32, device=c.device).view(torch.uint32)
    if int(c.min()) < 0 or int(c.max()) >= (1 << bits):
        raise PackError(f"codes out of range for {bits}-bit packing")
    c8 = c.to(torch.uint8).reshape(-1, 1)
    out = torch.empty(c.numel() * bits // 32, dtype=torch.int32, device=c.device)
    call("qigen_pack_rowseq", c8.data_ptr(), c8.shape[0], 1, bits, out.data_ptr(),
         _dev.stream_handle())
    return out.view(torch.uint32)


def unpack_words(words, bits: int) -> torch.Tensor:
    """packing.py:73-90."""
    _check_bits(bits)
    w = _as_words(words)
    if w.dim() != 1:
        raise PackError(f"words must be 1-D, got shape {tuple(w.shape)}")
    unit, kw = pack_unit(bits)
    if w.numel() % kw:
        raise PackError(f"word count {w.numel()} is not a multiple of {kw}")
    n = w.numel() // kw * unit
    out = torch.empty((n, 1), dtype=torch.uint8, device=w.device)
    if n:
        call("qigen_unpack_rowseq", w.data_ptr(), n, 1, bits, out.data_ptr(), _dev.stream_handle())
    return out[:, 0]


def _as_words(words) -> torch.Tensor:
    """uint32 words (numpy uint32 / torch uint32 / int32 view) -> CUDA int32 view."""
    if isinstance(words, torch.Tensor):
        t = words
        if t.dtype != torch.int32:
            t = t.view(torch.int32) if t.element_size() == 4 else t.to(torch.int64).to(torch.int32)
        return t.to(_dev.require_cuda()).contiguous()
    a = np.ascontiguousarray(np.asarray(words, dtype=np.uint32)).view(np.int32)
    return _dev.to_device(a, torch.int32)


def morton_index(row_block: int, col_block: int) -> int:
    """packing.py:103-107: row bits to even positions, column bits to odd."""
    if row_block < 0 or col_block < 0:
        raise PackError("block coordinates must be non-negative")
    out = 0
    for i in range(32):
        out |= ((row_block >> i) & 1) << (2 * i)
        out |= ((col_block >> i) & 1) << (2 * i + 1)
    return out


def block_order(row_blocks: int, col_blocks: int) -> list[tuple[int, int]]:
    """packing.py:110-114: grid coordinates in storage (Morton) order."""
    return sorted(((r, c) for r in range(row_blocks) for c in range(col_blocks)),
                  key=lambda rc: morton_index(*rc))


def _grid(n: int, m: int, plan: TilePlan) -> tuple[int, int]:
    return -(-n // plan.m_b), -(-m // plan.t_b)


def _check_plan_config(plan: TilePlan, config: QuantConfig) -> None:
    """packing.py:163-172."""
    unit, _ = pack_unit(config.bits)
    if plan.m_b % unit:
        raise PackError(f"plan m_b={plan.m_b} does not cover whole {config.bits}-bit packed "
                        f"words (needs a multiple of {unit})")
    if config.group_size is not None and plan.m_b % config.group_size:
        raise PackError(f"plan m_b={plan.m_b} splits quantization groups of size "
                        f"{config.group_size}")


def block_table(n: int, m: int, plan: TilePlan) -> torch.Tensor:
    rbs, cbs = _grid(n, m, plan)
    order = np.asarray(block_order(rbs, cbs), dtype=np.int32).reshape(-1)
    return _dev.to_device(order, torch.int32)


@dataclass
class PackedMatrix:
    """packing.py:117-156 — words hold exactly n*m*bits/32 uint32 in storage
    order; scales/zeros are the [G, m] parameter arrays."""

    words: torch.Tensor
    n: int
    m: int
    config: QuantConfig
    scales: torch.Tensor
    zeros: torch.Tensor
    plan: TilePlan
    layout: Layout = Layout.ZCURVE
    _exec_cache: object = field(default=None, repr=False, compare=False)

    @property
    def groups(self) -> int:
        return int(self.scales.shape[0])

    def word_count(self) -> int:
        return self.n * self.m * self.config.bits // 32

    def payload_bits(self) -> tuple[int, int, int]:
        g = self.groups
        return (self.config.bits * self.n * self.m, 32 * g * self.m,
                self.config.zero_bits() * g * self.m)

    def validate(self) -> None:
        if tuple(self.words.shape) != (self.word_count(),):
            raise PackError(f"word count {self.words.numel()} != {self.word_count()}")
        if tuple(self.scales.shape) != tuple(self.zeros.shape):
            raise PackError("scales/zeros shape mismatch")


def lay_out_blocks(cm: CodeMatrix, plan: TilePlan, layout: Layout = Layout.ZCURVE) -> PackedMatrix:
    """packing.py:217-226 on the GPU: pack row-sequentially, then permute into
    Morton-ordered blocks (ZCURVE)."""
    cm.validate()
    _check_plan_config(plan, cm.config)
    n, m, bits = cm.n, cm.m, cm.config.bits
    check_row_count(n, bits)
    codes = _dev.to_device(cm.codes, torch.uint8)
    nw = n * m * bits // 32
    rowseq = torch.empty(nw, dtype=torch.int32, device=codes.device)
    st = _dev.stream_handle()
    call("qigen_pack_rowseq", codes.data_ptr(), n, m, bits, rowseq.data_ptr(), st)
    words = rowseq
    if layout is Layout.ZCURVE:
        blk = block_table(n, m, plan)
        words = torch.empty_like(rowseq)
        call("qigen_permute_zcurve", rowseq.data_ptr(), words.data_ptr(), n, m, bits, plan.m_b,
             plan.t_b, blk.data_ptr(), blk.numel() // 2, 1, st)
    return PackedMatrix(words.view(torch.uint32), n, m, cm.config,
                        _dev.to_device(cm.scales, torch.float32),
                        _dev.to_device(cm.zeros, torch.float32), plan, layout)


def rowseq_words(pm) -> torch.Tensor:
    """Words of any (reference or ours) PackedMatrix in ROW_SEQUENTIAL order, on
    the GPU (inverse permutation, packing.py:233-235)."""
    words = _as_words(pm.words)
    if words.numel() != pm.n * pm.m * pm.config.bits // 32:
        raise PackError(f"word count {words.numel()} != {pm.n * pm.m * pm.config.bits // 32}")
    if Layout(pm.layout.value) is Layout.ROW_SEQUENTIAL:
        return words
    blk = block_table(pm.n, pm.m, pm.plan)
    out = torch.empty_like(words)
    call("qigen_permute_zcurve", words.data_ptr(), out.data_ptr(), pm.n, pm.m, pm.config.bits,
         pm.plan.m_b, pm.plan.t_b, blk.data_ptr(), blk.numel() // 2, 0, _dev.stream_handle())
    return out


def extract_codes(pm) -> CodeMatrix:
    """packing.py:229-242 on the GPU."""
    if hasattr(pm, "validate"):
        pm.validate()
    rs = rowseq_words(pm)
    codes = torch.empty((pm.n, pm.m), dtype=torch.uint8, device=rs.device)
    call("qigen_unpack_rowseq", rs.data_ptr(), pm.n, pm.m, pm.config.bits, codes.data_ptr(),
         _dev.stream_handle())
    return CodeMatrix(codes, _dev.to_device(pm.scales, torch.float32),
                      _dev.to_device(pm.zeros, torch.float32), _as_config(pm.config))


def _as_config(cfg) -> QuantConfig:
    """Accept the reference's QuantConfig (duck-typed) as well as ours."""
    if isinstance(cfg, QuantConfig):
        return cfg
    zm = getattr(cfg.zero_mode, "value", cfg.zero_mode)
    return QuantConfig(cfg.bits, cfg.group_size, zm)
