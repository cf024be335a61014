"""QIGW weight file: lossless round trip, file size,
distinct errors.  CPU-only: matrices are quantized and packed by the oracle."""

import numpy as np
import pytest
import torch

from oracle import qigen_oracle as orc
from paper_2307_03738_b200 import weightfile as wf
from paper_2307_03738_b200.config import QuantConfig, ZeroMode
from paper_2307_03738_b200.packing import Layout, PackedMatrix
from paper_2307_03738_b200.perfmodel import TilePlan


def _pm(K, N, bits, g, zero_mode="real32", layout=Layout.ZCURVE, seed=0):
    rng = np.random.default_rng(seed)
    w = rng.normal(0, 0.02, (K, N)).astype(np.float32)
    codes, s, z = orc.quantize_matrix(w, bits, g, zero_mode)
    mu, tu, m_b, t_b = orc.plan(bits, g, (K, N))
    words = orc.lay_out_words(codes, bits, m_b, t_b, layout is Layout.ZCURVE)
    pm = PackedMatrix(torch.from_numpy(words.view(np.int32)), K, N,
                      QuantConfig(bits, g, ZeroMode.coerce(zero_mode)), torch.from_numpy(s),
                      torch.from_numpy(z), TilePlan(mu, tu, m_b, t_b), layout)
    return pm, codes


CASES = [(256, 96, 4, 64, "real32", Layout.ZCURVE), (512, 40, 3, None, "real32", Layout.ZCURVE),
         (320, 17, 2, 32, "real32", Layout.ROW_SEQUENTIAL), (256, 64, 3, 32, "quantized", Layout.ZCURVE),
         (128, 33, 4, None, "quantized", Layout.ROW_SEQUENTIAL), (64, 8, 2, 16, "quantized", Layout.ZCURVE)]


@pytest.mark.parametrize("K,N,bits,g,zm,layout", CASES)
def test_round_trip_and_size(tmp_path, K, N, bits, g, zm, layout):
    pm, _ = _pm(K, N, bits, g, zm, layout, seed=K + N)
    path = tmp_path / "w.qigw"
    size = wf.write_weight_file(pm, path)
    assert size == path.stat().st_size
    back = wf.read_weight_file(path)
    assert (back.n, back.m, back.config, back.plan, back.layout) == (pm.n, pm.m, pm.config, pm.plan, pm.layout)
    assert np.array_equal(back.words.numpy().view(np.uint32), pm.words.numpy().view(np.uint32))
    assert np.array_equal(back.scales.numpy().view(np.uint32), pm.scales.numpy().view(np.uint32))
    assert np.array_equal(back.zeros.numpy(), pm.zeros.numpy())  # QUANTIZED: -0.0 stores as code 0
    if zm == "real32":
        assert np.array_equal(back.zeros.numpy().view(np.uint32), pm.zeros.numpy().view(np.uint32))
    # size = 64-byte header + each payload section (payload_bits) rounded up to 64 bytes
    wbits, sbits, zbits = pm.payload_bits()
    zbytes = zbits // 8 if zm == "real32" else -(-zbits // 32) * 4  # whole u32 words

    def c64(b):
        return -(-b // 64) * 64
    assert size == 64 + c64(sbits // 8) + c64(zbytes) + c64(wbits // 8)


def test_pack_codes_matches_pack_words():
    rng = np.random.default_rng(1)
    for bits in (2, 3, 4):
        codes = rng.integers(0, 1 << bits, 96).astype(np.uint8)
        w = wf._pack_codes(codes, bits)
        assert np.array_equal(w, orc.pack_words(codes, bits).astype("<u4"))
        assert np.array_equal(wf._unpack_codes(w, bits, 96), codes)


def test_distinct_errors(tmp_path):
    pm, _ = _pm(256, 64, 4, 128)
    path = tmp_path / "w.qigw"
    wf.write_weight_file(pm, path)
    data = bytearray(path.read_bytes())
    bad = bytearray(data)
    bad[100] ^= 0x01  # one payload byte
    (tmp_path / "c").write_bytes(bad)
    with pytest.raises(wf.ChecksumError):
        wf.read_weight_file(tmp_path / "c")
    bad = bytearray(data)
    bad[:4] = b"QIGX"
    (tmp_path / "m").write_bytes(bad)
    with pytest.raises(wf.BadMagicError):
        wf.read_weight_file(tmp_path / "m")
    bad = bytearray(data)
    bad[4] = 9
    (tmp_path / "v").write_bytes(bad)
    with pytest.raises(wf.VersionError):
        wf.read_weight_file(tmp_path / "v")
    (tmp_path / "t").write_bytes(bytes(data[:-10]))
    with pytest.raises(wf.TruncatedError):
        wf.read_weight_file(tmp_path / "t")
    (tmp_path / "h").write_bytes(bytes(data[:20]))
    with pytest.raises(wf.TruncatedError):
        wf.read_weight_file(tmp_path / "h")
    for cls in (wf.ChecksumError, wf.BadMagicError, wf.VersionError, wf.TruncatedError):
        assert issubclass(cls, wf.WeightFileError) and issubclass(cls, ValueError)


@pytest.mark.gpu
def test_load_panels_gemv(tmp_path):
    """QIGW file -> GPU panel layout -> qGEMV against the dense oracle."""
    pm, codes = _pm(1024, 300, 3, 64, seed=5)
    path = tmp_path / "w.qigw"
    wf.write_weight_file(pm, path)
    pw = wf.load_panels(path)
    x = np.random.default_rng(2).normal(0, 1, 1024).astype(np.float32)
    y = pw.gemv(torch.from_numpy(x).cuda()).cpu().numpy()
    yref = orc.qgemv_reference(codes, pm.scales.numpy(), pm.zeros.numpy(), x)
    assert np.abs(y - yref).max() / (1 + np.abs(yref).max()) <= 1e-5
