"""QIGW weight file: write / read a PackedMatrix (External
Interfaces SPEC.md:181).  The reference declares the format but ships no code
for it; this module implements it, plus a direct load into the
GPU panel layout.

Layout (all little-endian, header packed):

    magic "QIGW" | version u16 | bits u8 | zero_mode u8 | n u64 | m u64 |
    group_size u64 (0 = FULL_COLUMN) | layout u8 | m_b u32 | t_b u32 |
    m_u u16 | t_u u16 | payload length u64 | CRC32 of payload u32

The 57-byte header is zero-padded to 64 bytes; the payload follows: scales
(f32 [G, m]), zeros (REAL32: f32 [G, m]; QUANTIZED: b-bit codes packed like
`pack_words`), packed words (u32, storage order of the
layout), each section starting 64-byte aligned (zero padding).  The payload
length counts every section and its padding; the CRC32 (zlib polynomial)
covers the whole payload.  Hence the file size is
`64 + sum_i ceil64(section_i)` bytes, with section bits equal to
`PackedMatrix.payload_bits()` (packing.py:144-149) before padding.

Errors are distinct classes: BadMagicError, VersionError,
TruncatedError, ChecksumError (all WeightFileError, a ValueError).
"""

from __future__ import annotations

import struct
import zlib
from pathlib import Path

import numpy as np
import torch

from .config import QuantConfig, ZeroMode
from .packing import Layout, PackedMatrix
from .perfmodel import TilePlan

MAGIC = b"QIGW"
VERSION = 1
_HEADER = struct.Struct("<4sHBBQQQBIIHHQI")  # 57 bytes
HEADER_BYTES = 64
_ZERO_MODE = {ZeroMode.REAL32: 0, ZeroMode.QUANTIZED: 1}


class WeightFileError(ValueError):
    """A QIGW file could not be read."""


class BadMagicError(WeightFileError):
    pass


class VersionError(WeightFileError):
    pass


class TruncatedError(WeightFileError):
    pass


class ChecksumError(WeightFileError):
    pass


def _ceil64(n: int) -> int:
    return (n + 63) // 64 * 64


def _host(a) -> np.ndarray:
    if isinstance(a, torch.Tensor):
        return a.detach().cpu().numpy()
    return np.asarray(a)


def _pack_codes(codes: np.ndarray, bits: int) -> np.ndarray:
    """b-bit codes -> little-endian uint32 words, code j at bits [j*b, j*b+b)
    of the stream (the pack_words convention, incl. 3-bit straddles); the
    stream is zero-padded to whole words."""
    c = codes.astype(np.uint8).reshape(-1)
    bitplanes = ((c[:, None] >> np.arange(bits, dtype=np.uint8)) & 1).astype(np.uint8)
    stream = bitplanes.reshape(-1)
    stream = np.concatenate([stream, np.zeros((-len(stream)) % 32, np.uint8)])
    return np.packbits(stream, bitorder="little").view("<u4")


def _unpack_codes(words: np.ndarray, bits: int, count: int) -> np.ndarray:
    stream = np.unpackbits(words.astype("<u4").view(np.uint8), bitorder="little")
    planes = stream[: count * bits].reshape(count, bits).astype(np.uint8)
    return (planes << np.arange(bits, dtype=np.uint8)).sum(axis=1).astype(np.uint8)


def _sections(pm) -> list[bytes]:
    cfg = pm.config
    scales = _host(pm.scales).astype("<f4")
    zeros = _host(pm.zeros)
    if ZeroMode.coerce(cfg.zero_mode) is ZeroMode.QUANTIZED:
        zsec = _pack_codes(np.rint(zeros).astype(np.int64).clip(0, (1 << cfg.bits) - 1),
                           cfg.bits).tobytes()
    else:
        zsec = zeros.astype("<f4").tobytes()
    words = _host(pm.words).astype(np.int64, copy=False) & 0xFFFFFFFF
    return [scales.tobytes(), zsec, words.astype("<u4").tobytes()]


def write_weight_file(pm, path) -> int:
    """write `pm` (this package's or the reference's PackedMatrix)
    to `path`; returns the file size in bytes."""
    cfg = pm.config
    payload = bytearray()
    for sec in _sections(pm):
        payload += sec
        payload += b"\0" * (_ceil64(len(sec)) - len(sec))
    layout = pm.layout.value if hasattr(pm.layout, "value") else int(pm.layout)
    head = _HEADER.pack(MAGIC, VERSION, cfg.bits, _ZERO_MODE[ZeroMode.coerce(cfg.zero_mode)],
                        pm.n, pm.m, cfg.group_size or 0, layout, pm.plan.m_b, pm.plan.t_b,
                        pm.plan.m_u, pm.plan.t_u, len(payload), zlib.crc32(payload) & 0xFFFFFFFF)
    data = head + b"\0" * (HEADER_BYTES - len(head)) + bytes(payload)
    Path(path).write_bytes(data)
    return len(data)


def read_weight_file(path) -> PackedMatrix:
    """read a QIGW file back into a PackedMatrix (host tensors;
    `qgemv` / `runtime.exec_layout` move it to the GPU layout on first use)."""
    data = Path(path).read_bytes()
    if len(data) < _HEADER.size:
        if data[:4] != MAGIC[: len(data[:4])]:
            raise BadMagicError(f"{path}: not a QIGW file")
        raise TruncatedError(f"{path}: header truncated ({len(data)} bytes)")
    (magic, version, bits, zmode, n, m, group, layout, m_b, t_b, m_u, t_u, plen,
     crc) = _HEADER.unpack_from(data)
    if magic != MAGIC:
        raise BadMagicError(f"{path}: bad magic {magic!r}")
    if version != VERSION:
        raise VersionError(f"{path}: version {version}, this reader supports {VERSION}")
    if len(data) < HEADER_BYTES + plen:
        raise TruncatedError(f"{path}: payload truncated ({len(data) - HEADER_BYTES} of {plen} bytes)")
    payload = memoryview(data)[HEADER_BYTES:HEADER_BYTES + plen]
    if zlib.crc32(payload) & 0xFFFFFFFF != crc:
        raise ChecksumError(f"{path}: payload checksum mismatch")
    zero_mode = ZeroMode.QUANTIZED if zmode == 1 else ZeroMode.REAL32
    cfg = QuantConfig(bits, group or None, zero_mode)
    G = cfg.groups_for_rows(n)
    off = 0

    def take(nbytes):
        nonlocal off
        if off + nbytes > plen:
            raise TruncatedError(f"{path}: section overruns the payload")
        sec = payload[off:off + nbytes]
        off += _ceil64(nbytes)
        return sec

    scales = np.frombuffer(take(4 * G * m), "<f4").reshape(G, m).copy()
    if zero_mode is ZeroMode.QUANTIZED:
        nz_words = -(-(G * m * bits) // 32)
        zc = _unpack_codes(np.frombuffer(take(4 * nz_words), "<u4"), bits, G * m)
        zeros = zc.astype(np.float32).reshape(G, m)
    else:
        zeros = np.frombuffer(take(4 * G * m), "<f4").reshape(G, m).copy()
    nw = n * m * bits // 32
    words = np.frombuffer(take(4 * nw), "<u4").copy()
    pm = PackedMatrix(torch.from_numpy(words.view(np.int32)), n, m, cfg,
                      torch.from_numpy(scales), torch.from_numpy(zeros),
                      TilePlan(m_u, t_u, m_b, t_b), Layout(layout))
    pm.validate()
    return pm


def load_panels(path):
    """Read a QIGW file straight into the GPU panel layout (PanelWeights)."""
    from .runtime import PanelWeights
    return PanelWeights.from_packed(read_weight_file(path))
