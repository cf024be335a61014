"""Pin the CPU oracle against fixtures produced by the reference itself
(tests/golden/make_golden.py).  Integer outputs must be bit-exact; the C port
of the reference's generated kernel must reproduce the reference kernel's
float32 output bit-for-bit."""

import numpy as np
import pytest

from oracle import qigen_oracle as orc


def _bits_equal(a, b):
    a, b = np.asarray(a), np.asarray(b)
    return a.shape == b.shape and np.array_equal(a.view(np.uint32), b.view(np.uint32))


def test_quantize_bit_exact(golden_quant_pack):
    data, cases = golden_quant_pack
    for c in cases:
        k = c["key"]
        codes, s, z = orc.quantize_matrix(data[k + "_w"], c["bits"], c["g"], c["zero_mode"])
        assert np.array_equal(codes, data[k + "_codes"]), c
        assert _bits_equal(s, data[k + "_scales"]), c   # signed zeros included
        assert _bits_equal(z, data[k + "_zeros"]), c


def test_pack_rowseq_and_zcurve_bit_exact(golden_quant_pack):
    data, cases = golden_quant_pack
    for c in cases:
        k = c["key"]
        codes = data[k + "_codes"]
        assert np.array_equal(orc.pack_rowseq(codes, c["bits"]), data[k + "_rowseq"]), c
        zc = orc.lay_out_words(codes, c["bits"], c["m_b"], c["t_b"], True)
        assert np.array_equal(zc, data[k + "_zcurve"]), c
        rs = orc.words_to_rowseq(zc, c["n"], c["m"], c["bits"], c["m_b"], c["t_b"], True)
        assert np.array_equal(orc.unpack_rowseq(rs, c["n"], c["m"], c["bits"]), codes)


def test_plans_match_reference(golden_plans):
    for p in golden_plans:
        kw = dict(l1_bits=p.get("l1_bits", 262144), vregs=p.get("vregs", 16))
        if "error" in p:
            with pytest.raises(ValueError):
                orc.plan(p["bits"], p["g"], p["dims"], **kw)
        else:
            assert list(orc.plan(p["bits"], p["g"], p["dims"], **kw)) == p["plan"], p


def test_kats(golden_kats):
    k = golden_kats
    c, s, z = orc.quantize_matrix(np.arange(16, dtype=np.float32)[:, None], 4, None)
    assert c[:, 0].tolist() == k["q_0_15"]["codes"] and s[0, 0] == k["q_0_15"]["s"]
    assert np.signbit(z[0, 0]) == k["q_0_15"]["z_signbit"]
    c, s, z = orc.quantize_matrix(np.full((8, 1), 0.37, np.float32), 4, None)
    assert c[:, 0].tolist() == k["q_const"]["codes"] and z[0, 0] == np.float32(k["q_const"]["z"])
    c, s, z = orc.quantize_matrix(np.array([[-1.0], [1.0]], np.float32), 2, None)
    assert c[:, 0].tolist() == k["q_pm1_b2"]["codes"] and s[0, 0] == np.float32(k["q_pm1_b2"]["s"])
    c, s, z = orc.quantize_matrix(np.array([[-1.0], [1.0]], np.float32), 2, None, "quantized")
    assert c[:, 0].tolist() == k["q_pm1_b2_quant"]["codes"] and z[0, 0] == k["q_pm1_b2_quant"]["z"]
    c, s, z = orc.quantize_matrix(np.full((4, 1), 0.37, np.float32), 4, None, "quantized")
    assert np.signbit(z[0, 0]) == k["q_const_quant"]["z_signbit"]
    c, s, z = orc.quantize_matrix(np.array([[0.0], [0.5], [3.0]], np.float32), 2, None)
    assert c[:, 0].tolist() == k["q_tie_b2"]["codes"]
    assert int(orc.pack_words(np.arange(1, 9), 4)[0]) == k["pack_4"] == 0x87654321
    assert orc.pack_words(np.full(32, 7), 3).tolist() == k["pack_3_all7"]
    assert orc.pack_words(np.array([1] + [0] * 31), 3).tolist() == k["pack_3_one"]
    assert int(orc.pack_words(np.tile(np.arange(4), 4), 2)[0]) == k["pack_2"] == 0xE4E4E4E4
    for key, v in k["morton"].items():
        r, cc = map(int, key.split(","))
        assert orc.morton_index(r, cc) == v
    assert [list(t) for t in orc.block_order(2, 2)] == k["block_order_2x2"]


@pytest.mark.parametrize("bits", [2, 3, 4])
def test_pack_unpack_inverse_random(bits):
    rng = np.random.default_rng(bits)
    unit = orc.pack_unit(bits)[0]
    codes = rng.integers(0, 1 << bits, size=unit * 10_000).astype(np.uint8)
    assert np.array_equal(orc.unpack_words(orc.pack_words(codes, bits), bits), codes)


def test_qgemv_port_bit_exact_vs_reference_kernel(golden_qgemv):
    data, cases = golden_qgemv
    for c in cases:
        k = c["key"]
        codes, s, z = orc.quantize_matrix(data[k + "_w"], c["bits"], c["g"])
        ex = orc.ExecLayout(orc.pack_rowseq(codes, c["bits"]), s, z, c["n"], c["m"],
                            c["bits"], c["g"], c["m_b"], c["t_b"])
        assert _bits_equal(ex.xsums(ex.pad_x(data[k + "_x"])), data[k + "_xsums"])
        for threads in (1, 3):   # thread-count invariance
            y = orc.qgemv_port(ex, data[k + "_x"], threads=threads)
            assert _bits_equal(y, data[k + "_y"]), (c, threads)
        yd = orc.qgemv_reference(codes, s, z, data[k + "_x"])
        assert np.abs(yd - data[k + "_y"]).max() / (1 + np.abs(yd).max()) <= 1e-5
