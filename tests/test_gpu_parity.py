"""GPU parity: the CUDA path (through the C ABI) against the CPU oracle and the
reference-generated golden fixtures.  Integer outputs bit-exact; qgemv within
the reference's own tolerance |dy|_inf / (1 + |y|_inf) <= 1e-5
for f32 activations."""

import numpy as np
import pytest
import torch

from oracle import qigen_oracle as orc

pytestmark = pytest.mark.gpu

TOL = 1e-5        # SPEC.md:369 (f32 x)
TOL_HALF = 1e-5   # f16/bf16 x: compared against an oracle fed the same rounded x


@pytest.fixture(scope="module")
def q():
    assert torch.cuda.is_available(), "GPU tests need a CUDA device"
    import paper_2307_03738_b200 as q
    q._lib.lib()
    return q


def rel_err(y, yref):
    y, yref = np.asarray(y, np.float64), np.asarray(yref, np.float64)
    return np.abs(y - yref).max() / (1.0 + np.abs(yref).max())


def bits_equal(a, b):
    a, b = np.asarray(a), np.asarray(b)
    return a.shape == b.shape and np.array_equal(a.view(np.uint32), b.view(np.uint32))


# --- quantize / pack: bit-exact against reference fixtures --------------------

def test_quantize_bit_exact_vs_reference(q, golden_quant_pack):
    data, cases = golden_quant_pack
    for c in cases:
        k = c["key"]
        cm = q.quantize_matrix(data[k + "_w"], q.QuantConfig(c["bits"], c["g"], c["zero_mode"]))
        codes, s, z = cm.numpy()
        assert np.array_equal(codes, data[k + "_codes"]), c
        assert bits_equal(s, data[k + "_scales"]), c
        assert bits_equal(z, data[k + "_zeros"]), c


def test_pack_bit_exact_vs_reference(q, golden_quant_pack):
    data, cases = golden_quant_pack
    for c in cases:
        k = c["key"]
        cfg = q.QuantConfig(c["bits"], c["g"], c["zero_mode"])
        cm = q.quantize_matrix(data[k + "_w"], cfg)
        plan = q.TilePlan(3, 3, c["m_b"], c["t_b"])
        pr = q.lay_out_blocks(cm, plan, q.Layout.ROW_SEQUENTIAL)
        pz = q.lay_out_blocks(cm, plan, q.Layout.ZCURVE)
        assert np.array_equal(pr.words.cpu().numpy(), data[k + "_rowseq"]), c
        assert np.array_equal(pz.words.cpu().numpy(), data[k + "_zcurve"]), c
        back = q.extract_codes(pz)
        assert np.array_equal(back.codes.cpu().numpy(), data[k + "_codes"]), c


def test_kats_on_gpu(q, golden_kats):
    k = golden_kats
    codes, p = q.quantize_group(np.arange(16, dtype=np.float32), 4)
    assert codes.cpu().tolist() == k["q_0_15"]["codes"] and p.scale == 1.0
    assert np.signbit(p.zero) == k["q_0_15"]["z_signbit"]
    codes, p = q.quantize_group(np.array([-1, 1], np.float32), 2)
    assert codes.cpu().tolist() == k["q_pm1_b2"]["codes"] and p.zero == k["q_pm1_b2"]["z"]
    codes, p = q.quantize_group(np.array([-1, 1], np.float32), 2, "quantized")
    assert codes.cpu().tolist() == k["q_pm1_b2_quant"]["codes"] and p.zero == 1.0
    codes, p = q.quantize_group(np.full(4, 0.37, np.float32), 4, "quantized")
    assert np.signbit(p.zero) == k["q_const_quant"]["z_signbit"]
    codes, p = q.quantize_group(np.array([0, 0.5, 3], np.float32), 2)
    assert codes.cpu().tolist() == k["q_tie_b2"]["codes"]
    assert int(q.pack_words(np.arange(1, 9), 4).cpu().numpy()[0]) == k["pack_4"]
    assert q.pack_words(np.full(32, 7), 3).cpu().numpy().tolist() == k["pack_3_all7"]
    assert q.pack_words(np.array([1] + [0] * 31), 3).cpu().numpy().tolist() == k["pack_3_one"]
    assert int(q.pack_words(np.tile(np.arange(4), 4), 2).cpu().numpy()[0]) == k["pack_2"]
    with pytest.raises(q.PackError):
        q.pack_words(np.array([16] + [0] * 7), 4)
    with pytest.raises(q.PackError):
        q.pack_words(np.zeros(7), 4)
    with pytest.raises(q.ConfigError):
        q.quantize_matrix(np.full((4, 4), np.nan, np.float32), q.QuantConfig(4, None))
    with pytest.raises(q.ConfigError):
        q.quantize_matrix(np.zeros((100, 4), np.float32), q.QuantConfig(4, 64))


@pytest.mark.parametrize("bits", [2, 3, 4])
def test_pack_unpack_inverse_random(q, bits):
    rng = np.random.default_rng(bits)
    unit = q.pack_unit(bits)[0]
    codes = rng.integers(0, 1 << bits, size=unit * 10_000).astype(np.uint8)
    w = q.pack_words(codes, bits)
    assert np.array_equal(w.cpu().numpy(), orc.pack_words(codes, bits))
    assert np.array_equal(q.unpack_words(w, bits).cpu().numpy(), codes)


@pytest.mark.parametrize("shape", [(4096, 4096), (4096, 11008), (11008, 4096)])
def test_quantize_bit_exact_large(q, shape):
    """BASELINE configs[1] shapes (4096^2, 4096x11008, 11008x4096) at every
    (b, g): codes, scales, zeros, ROW_SEQUENTIAL and ZCURVE words bit-exact
    against the oracle."""
    K, N = shape
    rng = np.random.default_rng(7 + K + 3 * N)
    w = rng.normal(0, 0.02, (K, N)).astype(np.float32)
    for bits in (2, 3, 4):
        for g in (32, 64, 128, None):
            cm = q.quantize_matrix(w, q.QuantConfig(bits, g))
            codes, s, z = cm.numpy()
            rc, rs, rz = orc.quantize_matrix(w, bits, g)
            assert np.array_equal(codes, rc), (K, N, bits, g)
            assert bits_equal(s, rs) and bits_equal(z, rz), (K, N, bits, g)
            p = q.plan(q.DEFAULT_HARDWARE, cm.config, (K, N))
            rowseq = q.lay_out_blocks(cm, p, q.Layout.ROW_SEQUENTIAL).words.cpu().numpy()
            assert np.array_equal(rowseq, orc.pack_rowseq(rc, bits)), (K, N, bits, g)
            zc = q.lay_out_blocks(cm, p, q.Layout.ZCURVE).words.cpu().numpy()
            assert np.array_equal(zc, orc.lay_out_words(rc, bits, p.m_b, p.t_b, True)), \
                (K, N, bits, g)


# --- panel layout ---------------------------------------------------------------

@pytest.mark.parametrize("bits", [2, 3, 4])
@pytest.mark.parametrize("shape", [(256, 16), (4096, 4096), (320, 40), (11008, 48), (96, 8)])
def test_panel_layout_round_trip(q, bits, shape):
    n, m = shape
    if n % q.pack_unit(bits)[0]:
        pytest.skip("row count not a packing unit multiple")
    rng = np.random.default_rng(n + m + bits)
    codes = rng.integers(0, 1 << bits, size=(n, m)).astype(np.uint8)
    cm = q.CodeMatrix(torch.from_numpy(codes).cuda(), torch.ones(1, m).cuda(),
                      torch.zeros(1, m).cuda(), q.QuantConfig(bits, None))
    pw = q.PanelWeights.from_codes(cm)
    assert np.array_equal(pw.to_codes().cpu().numpy(), codes)
    # and via reference words (ROW_SEQUENTIAL and ZCURVE)
    pm = q.lay_out_blocks(cm, q.plan(q.DEFAULT_HARDWARE, cm.config, (n, m)), q.Layout.ZCURVE)
    pw2 = q.PanelWeights.from_packed(pm)
    assert torch.equal(pw2.qw, pw.qw)


# --- qgemv ------------------------------------------------------------------------

def _case(q, K, N, bits, g, seed=0, zero_mode="real32"):
    rng = np.random.default_rng(seed)
    w = rng.normal(0, 0.02, (K, N)).astype(np.float32)
    cfg = q.QuantConfig(bits, g, zero_mode)
    cm = q.quantize_matrix(w, cfg)
    codes, s, z = cm.numpy()
    return cm, codes, s, z, rng


def test_qgemv_vs_reference_kernel_golden(q, golden_qgemv):
    """Against the outputs of the reference's own generated kernels."""
    data, cases = golden_qgemv
    assert any(c["g"] == 16 for c in cases)
    for c in cases:  # every fixture, g = 16 included
        k = c["key"]
        cfg = q.QuantConfig(c["bits"], c["g"])
        cm = q.quantize_matrix(data[k + "_w"], cfg)
        pm = q.lay_out_blocks(cm, q.TilePlan(3, 3, c["m_b"], c["t_b"]))
        y = q.qgemv(pm, data[k + "_x"])
        assert rel_err(y, data[k + "_y"]) <= TOL, c


SWEEP = [(b, g, shp) for b in (2, 3, 4) for g in (32, 64, 128, None)
         for shp in [(4096, 4096), (4096, 11008), (11008, 4096)]]


@pytest.mark.parametrize("bits,g,shape", SWEEP)
def test_qgemv_sweep_vs_oracle(q, bits, g, shape):
    """BASELINE configs[1]: every (b, g, shape) vs the dense fp64 oracle."""
    K, N = shape
    cm, codes, s, z, rng = _case(q, K, N, bits, g, seed=bits * 7 + (g or 0))
    pw = q.PanelWeights.from_codes(cm)
    x = rng.normal(0, 1, K).astype(np.float32)
    y = pw.gemv(torch.from_numpy(x).cuda()).cpu().numpy()
    yref = orc.qgemv_reference(codes, s, z, x)
    assert rel_err(y, yref) <= TOL, (bits, g, shape, rel_err(y, yref))


def test_qgemv_cfg0_vs_port_and_dense(q):
    """configs[0]: 4096^2 b4 g128 — GPU vs the C port of the reference kernel
    (same exec layout as the reference) and the dense oracle."""
    K = N = 4096
    cm, codes, s, z, rng = _case(q, K, N, 4, 128, seed=0)
    x = rng.normal(0, 1, K).astype(np.float32)
    p = q.plan(q.DEFAULT_HARDWARE, cm.config, (K, N))
    pm = q.lay_out_blocks(cm, p)
    y = q.qgemv(pm, x)
    ex = orc.ExecLayout(orc.pack_rowseq(codes, 4), s, z, K, N, 4, 128, p.m_b, p.t_b)
    yport = orc.qgemv_port(ex, x, threads=4)
    yref = orc.qgemv_reference(codes, s, z, x)
    assert rel_err(y, yref) <= TOL and rel_err(yport, yref) <= TOL
    assert rel_err(y, yport) <= TOL


@pytest.mark.parametrize("tokens", [1, 2, 3, 4, 8, 16])
def test_qgemv_small_batch(q, tokens):
    K, N = 2048, 1536
    cm, codes, s, z, rng = _case(q, K, N, 4, 64, seed=tokens)
    pw = q.PanelWeights.from_codes(cm)
    X = rng.normal(0, 1, (tokens, K)).astype(np.float32)
    # the exact IMMA path at every token count
    Y = pw.gemv(torch.from_numpy(X).cuda(), path="gemv").cpu().numpy()
    for t in range(tokens):
        yref = orc.qgemv_reference(codes, s, z, X[t])
        assert rel_err(Y[t], yref) <= TOL, (tokens, t)


@pytest.mark.parametrize("dtype", [torch.float16, torch.bfloat16])
def test_qgemv_half_activations(q, dtype):
    K, N = 4096, 1024
    cm, codes, s, z, rng = _case(q, K, N, 4, 128, seed=3)
    pw = q.PanelWeights.from_codes(cm)
    xh = torch.from_numpy(rng.normal(0, 1, K).astype(np.float32)).to(dtype)
    y = pw.gemv(xh.cuda()).cpu().numpy()
    yref = orc.qgemv_reference(codes, s, z, xh.float().numpy())
    assert rel_err(y, yref) <= TOL_HALF


@pytest.mark.parametrize("shape", [(32, 8), (96, 24), (288, 40), (544, 1000), (1024, 17)])
@pytest.mark.parametrize("bits", [2, 3, 4])
def test_qgemv_ragged_shapes(q, shape, bits):
    """K not a multiple of 256, N not a multiple of 16 (padding paths)."""
    K, N = shape
    if K % q.pack_unit(bits)[0]:
        pytest.skip("K must fill packing units")
    for g in (32, None):
        if g and K % g:
            continue
        cm, codes, s, z, rng = _case(q, K, N, bits, g, seed=K + N)
        pm = q.lay_out_blocks(cm, q.plan(q.DEFAULT_HARDWARE, cm.config, (K, N)))
        x = rng.normal(0, 1, K).astype(np.float32)
        assert rel_err(q.qgemv(pm, x), orc.qgemv_reference(codes, s, z, x)) <= TOL


def test_acceptance_1_oracle_equivalence(q):
    """SPEC acceptance #1: every bits in {2,3,4} x grouping in
    {16, 32, 64, 128, FULL_COLUMN} on 20 random shapes with n, m <= 1024: qgemv
    matches qgemv_reference within relative max-norm 1e-5."""
    rng = np.random.default_rng(454)
    for bits in (2, 3, 4):
        unit = q.pack_unit(bits)[0]
        for g in (16, 32, 64, 128, None):
            step = unit if g is None else int(np.lcm(unit, g))
            for _ in range(20):
                K = int(rng.integers(1, 1024 // step + 1)) * step
                N = int(rng.integers(1, 1025))
                w = rng.normal(0, 0.02, (K, N)).astype(np.float32)
                codes, s, z = orc.quantize_matrix(w, bits, g)
                cm = q.quantize_matrix(w, q.QuantConfig(bits, g))
                pm = q.lay_out_blocks(cm, q.plan(q.DEFAULT_HARDWARE, cm.config, (K, N)))
                x = rng.normal(0, 1, K).astype(np.float32)
                err = rel_err(q.qgemv(pm, x), orc.qgemv_reference(codes, s, z, x))
                assert err <= TOL, (bits, g, K, N, err)


def test_acceptance_6_thread_invariance(q):
    """SPEC acceptance #6: qgemv output bit-identical for threads = 1, 2, 4, 8
    (`threads` has no GPU meaning; the kernel's reduction order is fixed)."""
    rng = np.random.default_rng(6)
    for K, N, bits, g in [(1024, 1000, 4, 64), (768, 333, 3, None), (512, 64, 2, 16)]:
        cm = q.quantize_matrix(rng.normal(0, 0.02, (K, N)).astype(np.float32),
                               q.QuantConfig(bits, g))
        pm = q.lay_out_blocks(cm, q.plan(q.DEFAULT_HARDWARE, cm.config, (K, N)))
        x = rng.normal(0, 1, K).astype(np.float32)
        ys = [q.qgemv(pm, x, threads=t) for t in (1, 2, 4, 8)]
        assert all(np.array_equal(ys[0], y) for y in ys[1:])


@pytest.mark.parametrize("bits", [2, 3, 4])
@pytest.mark.parametrize("shape", [(4096, 4096), (4096, 11008), (11008, 4096), (352, 1000)])
def test_qgemv_group16(q, bits, shape):
    """g = 16 (two groups per m16n8k32 step: k16 IMMAs, a flush per half step)
    at BASELINE shapes and a ragged one: 1 / 3 / 8 tokens, the forced prep-kernel
    path and the RMSNorm prologue, against the oracle."""
    from paper_2307_03738_b200 import _lib
    K, N = shape
    if K % q.pack_unit(bits)[0]:
        pytest.skip("K must fill packing units")
    cm, codes, s, z, rng = _case(q, K, N, bits, 16, seed=K + bits)
    pw = q.PanelWeights.from_codes(cm)
    for tokens in (1, 3, 8):
        X = rng.normal(0, 1, (tokens, K)).astype(np.float32)
        ref = orc.qgemv_reference(codes, s, z, X)
        Y = pw.gemv(torch.from_numpy(X).cuda()).cpu().numpy()
        assert rel_err(Y, ref) <= TOL, (tokens, rel_err(Y, ref))
    try:
        _lib.lib().qigen_debug_force_prep(1)
        Yp = pw.gemv(torch.from_numpy(X).cuda()).cpu().numpy()
    finally:
        _lib.lib().qigen_debug_force_prep(0)
    assert rel_err(Yp, ref) <= TOL
    wn = rng.uniform(0.5, 1.5, K).astype(np.float32)
    Yn = pw.gemv(torch.from_numpy(X).cuda(), prologue="rmsnorm",
                 norm_weight=torch.from_numpy(wn).cuda()).cpu().numpy()
    for t in range(tokens):
        xn = X[t] / np.sqrt(np.mean(X[t].astype(np.float64) ** 2) + 1e-5) * wn
        assert rel_err(Yn[t], orc.qgemv_reference(codes, s, z, xn)) <= TOL


def test_qgemv_batch_with_group16(q):
    """qgemv_batch over a list mixing g = 16 (single GEMVs after the grouped
    launch) with grouped-kernel configs, host and device inputs."""
    pms, xs, refs = [], [], []
    for i, (K, N, b, g) in enumerate([(1024, 512, 4, 16), (2048, 300, 3, 32), (512, 100, 2, 16),
                                      (768, 640, 4, None)]):
        cm, codes, s, z, rng = _case(q, K, N, b, g, seed=90 + i)
        pms.append(q.lay_out_blocks(cm, q.plan(q.DEFAULT_HARDWARE, cm.config, (K, N))))
        xs.append(rng.normal(0, 1, K).astype(np.float32))
        refs.append(orc.qgemv_reference(codes, s, z, xs[-1]))
    for _ in range(2):
        for y, r in zip(q.qgemv_batch(pms, xs), refs):
            assert rel_err(y, r) <= TOL
    for y, r in zip(q.qgemv_batch(pms, [torch.from_numpy(x).cuda() for x in xs]), refs):
        assert rel_err(y.cpu().numpy(), r) <= TOL
    only16 = [pms[0], pms[2]]
    for y, r in zip(q.qgemv_batch(only16, [xs[0], xs[2]]), [refs[0], refs[2]]):
        assert rel_err(y, r) <= TOL


def test_qgemv_properties(q):
    K, N = 4096, 2048
    cm, codes, s, z, rng = _case(q, K, N, 3, 64, seed=11)
    pw = q.PanelWeights.from_codes(cm)
    x1 = torch.from_numpy(rng.normal(0, 1, K).astype(np.float32)).cuda()
    x2 = torch.from_numpy(rng.normal(0, 1, K).astype(np.float32)).cuda()
    # zero in -> zero out, exactly
    assert torch.count_nonzero(pw.gemv(torch.zeros(K, device="cuda"))) == 0
    # determinism: repeated calls bit-identical
    a, b = pw.gemv(x1), pw.gemv(x1)
    assert torch.equal(a, b)
    # any K split gives the same answer within tolerance
    for ks in (1, 2, 3, 8):
        assert rel_err(pw.gemv(x1, k_splits=ks).cpu(), a.cpu()) <= 1e-6
    # linearity
    lhs = pw.gemv(2.0 * x1 - 0.5 * x2).cpu().numpy()
    rhs = (2.0 * a - 0.5 * pw.gemv(x2)).cpu().numpy()
    assert np.abs(lhs - rhs).max() / (1 + np.abs(rhs).max()) <= 1e-4
    # accumulate into y
    y = pw.gemv(x1)
    pw.gemv(x2, out=y.view(1, -1), accumulate=True)
    assert rel_err(y.cpu(), (a + pw.gemv(x2)).cpu()) <= 1e-6


def test_grouped_g_equals_n_vs_full_column(q):
    """Acceptance #8: GROUPED(g=n) == FULL_COLUMN within 1e-6."""
    rng = np.random.default_rng(5)
    for _ in range(3):
        K, N = 1024, 512
        w = rng.normal(0, 0.02, (K, N)).astype(np.float32)
        x = rng.normal(0, 1, K).astype(np.float32)
        yg = q.PanelWeights.from_float(w, q.QuantConfig(4, K)).gemv(torch.from_numpy(x).cuda())
        yf = q.PanelWeights.from_float(w, q.QuantConfig(4, None)).gemv(torch.from_numpy(x).cuda())
        assert rel_err(yg.cpu(), yf.cpu()) <= 1e-6


def test_qgemv_accepts_reference_style_packed_matrix(q):
    """A reference PackedMatrix carries numpy words and numpy params."""
    from types import SimpleNamespace
    K, N = 512, 96
    cm, codes, s, z, rng = _case(q, K, N, 3, 64, seed=2)
    p = q.plan(q.DEFAULT_HARDWARE, cm.config, (K, N))
    words = orc.lay_out_words(codes, 3, p.m_b, p.t_b, True)
    ref_like = SimpleNamespace(words=words, n=K, m=N, config=cm.config, scales=s, zeros=z,
                               plan=p, layout=q.Layout.ZCURVE, _exec_cache=None)
    x = rng.normal(0, 1, K).astype(np.float32)
    y = q.qgemv(ref_like, x, orc.input_sums(x, 64), threads=4)
    assert rel_err(y, orc.qgemv_reference(codes, s, z, x)) <= TOL
    assert ref_like._exec_cache is not None
    with pytest.raises(q.ConfigError):
        q.qgemv(ref_like, x, threads=0)


def test_input_sums_and_dense_reference(q):
    rng = np.random.default_rng(9)
    x = rng.normal(0, 1, 4096).astype(np.float32)
    sums = q.input_sums(x, 64)
    assert np.allclose(sums.per_group.cpu().numpy(), orc.input_sums(x, 64), rtol=0, atol=1e-5)
    assert abs(sums.total - float(orc.input_sums(x, None)[0])) <= 1e-4
    ones = q.input_sums(np.ones(64, np.float32), 16)
    assert ones.per_group.cpu().tolist() == [16.0] * 4 and ones.total == 64.0
    cm, codes, s, z, rng = _case(q, 256, 64, 4, 32, seed=1)
    pm = q.lay_out_blocks(cm, q.plan(q.DEFAULT_HARDWARE, cm.config, (256, 64)))
    yd = q.qgemv_reference(pm, x[:256])
    assert np.allclose(yd, orc.qgemv_reference(codes, s, z, x[:256]), rtol=1e-12, atol=1e-12)


@pytest.mark.parametrize("tokens", [1, 3, 8])
@pytest.mark.parametrize("bits,g", [(4, 128), (3, 64), (2, 32), (4, None), (3, 512)])
def test_qgemv_prep_kernel_path(q, tokens, bits, g):
    """Activation digits from the separate prep kernel (forced) vs the oracle,
    including the fused RMSNorm / SwiGLU prologues."""
    from paper_2307_03738_b200 import _lib
    K, N = 2048, 640
    cm, codes, s, z, rng = _case(q, K, N, bits, g, seed=tokens + bits)
    pw = q.PanelWeights.from_codes(cm)
    X = rng.normal(0, 1, (tokens, K)).astype(np.float32)
    try:
        _lib.lib().qigen_debug_force_prep(1)
        Y = pw.gemv(torch.from_numpy(X).cuda()).cpu().numpy()
        wn = rng.uniform(0.5, 1.5, K).astype(np.float32)
        Yn = pw.gemv(torch.from_numpy(X).cuda(), prologue="rmsnorm",
                     norm_weight=torch.from_numpy(wn).cuda()).cpu().numpy()
        GU = rng.normal(0, 1, (tokens, 2 * K)).astype(np.float32)
        Ys = pw.gemv(torch.from_numpy(GU).cuda(), prologue="swiglu").cpu().numpy()
    finally:
        _lib.lib().qigen_debug_force_prep(0)
    Yn_fused = pw.gemv(torch.from_numpy(X).cuda(), prologue="rmsnorm",
                       norm_weight=torch.from_numpy(wn).cuda()).cpu().numpy()
    for t in range(tokens):
        assert rel_err(Y[t], orc.qgemv_reference(codes, s, z, X[t])) <= TOL
        xn = X[t] / np.sqrt(np.mean(X[t].astype(np.float64) ** 2) + 1e-5) * wn
        assert rel_err(Yn[t], orc.qgemv_reference(codes, s, z, xn)) <= 1e-5
        assert rel_err(Yn_fused[t], orc.qgemv_reference(codes, s, z, xn)) <= 1e-5
        g_, u_ = GU[t, :K].astype(np.float64), GU[t, K:].astype(np.float64)
        xs = g_ / (1 + np.exp(-g_)) * u_
        assert rel_err(Ys[t], orc.qgemv_reference(codes, s, z, xs)) <= 1e-5


TOL_TC = 2e-3  # tensor-core path: fp16 dequantized weights x fp16 activations, f32 accumulate


@pytest.mark.parametrize("tokens", [16, 17, 33, 64, 100])
@pytest.mark.parametrize("g", [32, 64, 128, 256])
def test_small_batch_tensor_core_path(q, tokens, g):
    """BASELINE configs[2] path (M >= 16): tcgen05 kernel vs the fp64 dense
    oracle (and vs the exact IMMA path), ragged N and token counts."""
    K, N = 2048, 1040
    cm, codes, s, z, rng = _case(q, K, N, 4, g, seed=tokens + g)
    pw = q.PanelWeights.from_codes(cm)
    X = rng.normal(0, 1, (tokens, K)).astype(np.float32)
    xt = torch.from_numpy(X).cuda()
    Y = pw.gemv(xt).cpu().numpy()
    ref = np.stack([orc.qgemv_reference(codes, s, z, X[t]) for t in range(tokens)])
    assert rel_err(Y, ref) <= TOL_TC
    Y2 = pw.gemv(xt, path="gemv").cpu().numpy()
    assert rel_err(Y2, ref) <= TOL
    # accumulate into y and fp16 activations
    Yacc = torch.from_numpy(Y).cuda()
    pw.gemv(xt, out=Yacc, accumulate=True)
    assert rel_err(Yacc.cpu().numpy(), 2 * ref) <= TOL_TC
    Yh = pw.gemv(xt.half()).cpu().numpy()
    refh = np.stack([orc.qgemv_reference(codes, s, z, X[t].astype(np.float16).astype(np.float32))
                     for t in range(tokens)])
    assert rel_err(Yh, refh) <= TOL_TC


@pytest.mark.parametrize("M", [1, 4, 16, 64])
def test_cfg2_shapes_vs_oracle(q, M):
    """configs[2]: K = N = 8192, 4-bit g64, M in {1, 4, 16, 64} against the CPU
    oracle's dense fp64 product (oracle quantize, not the GPU's own dequantize).
    The exact IMMA GEMV (SIMT path below 16 tokens) at 1e-5 for every M; the
    tcgen05 path (auto from 16 tokens) at TOL_TC."""
    K = N = 8192
    rng = np.random.default_rng(99 + M)
    w = rng.normal(0, 0.02, (K, N)).astype(np.float32)
    codes, s, z = orc.quantize_matrix(w, 4, 64)
    cm = q.quantize_matrix(w, q.QuantConfig(4, 64))
    pm = q.lay_out_blocks(cm, q.plan(q.DEFAULT_HARDWARE, cm.config, (K, N)))
    X = rng.normal(0, 1, (M, K)).astype(np.float32)
    ref = orc.qgemv_reference(codes, s, z, X)  # [M, N] fp64
    Y = q.qgemv(pm, X)                          # the public seam, host in / host out
    assert Y.shape == (M, N)
    assert rel_err(Y, ref) <= (TOL if M < 16 else TOL_TC), M
    pw = q.runtime.exec_layout(pm)
    Yg = pw.gemv(torch.from_numpy(X).cuda(), path="gemv").cpu().numpy()
    assert rel_err(Yg, ref) <= TOL, M


@pytest.mark.parametrize("bits,g", [(4, 128), (3, 64), (2, 32), (4, None)])
def test_qgemv_quantized_zero_mode(q, bits, g):
    """ZeroMode.QUANTIZED (zeros rounded to codes, quant.py:88-90) through the
    qgemv seam, the grouped launch and 2 tokens, vs the oracle."""
    K, N = 4096, 1000
    cm, codes, s, z, rng = _case(q, K, N, bits, g, seed=bits + (g or 0), zero_mode="quantized")
    w = np.random.default_rng(bits + (g or 0)).normal(0, 0.02, (K, N)).astype(np.float32)
    oc, os_, oz = orc.quantize_matrix(w, bits, g, "quantized")  # the same W as _case
    assert np.array_equal(codes, oc) and bits_equal(s, os_) and bits_equal(z, oz)
    assert np.all(z == np.round(z))  # integer zero points
    pm = q.lay_out_blocks(cm, q.plan(q.DEFAULT_HARDWARE, cm.config, (K, N)))
    X = rng.normal(0, 1, (2, K)).astype(np.float32)
    ref = orc.qgemv_reference(codes, s, z, X)
    assert rel_err(q.qgemv(pm, X[0]), ref[0]) <= TOL
    assert rel_err(q.qgemv(pm, X), ref) <= TOL
    (yb,) = q.qgemv_batch([pm], [X[1]])
    assert rel_err(yb, ref[1]) <= TOL


# --- grouped GEMV (independent GEMVs in one persistent launch) ----------------

def _group_cases(q, specs, seed=0, dtype=torch.float32, tokens=1):
    from paper_2307_03738_b200.runtime import GemvGroup
    entries, refs = [], []
    for i, (K, N, bits, g) in enumerate(specs):
        cm, codes, s, z, rng = _case(q, K, N, bits, g, seed=seed + i)
        pw = q.PanelWeights.from_codes(cm)
        X = torch.from_numpy(rng.normal(0, 1, (tokens, K)).astype(np.float32)).to(dtype)
        y = torch.full((tokens, N), float("nan"), device="cuda")
        entries.append((pw, X.cuda(), y))
        refs.append([orc.qgemv_reference(codes, s, z, X[t].float().numpy()) for t in range(tokens)])
    return GemvGroup(entries), entries, refs


def test_group_gemv_sweep_vs_oracle(q):
    """BASELINE configs[1] mix (all b x g, the three shapes) in one launch."""
    specs = [(K, N, b, g) for (K, N) in [(4096, 4096), (4096, 11008), (11008, 4096)]
             for b in (2, 3, 4) for g in (32, 64, 128, None)]
    grp, entries, refs = _group_cases(q, specs)
    grp.run()
    torch.cuda.synchronize()
    for (pw, x, y), r, spec in zip(entries, refs, specs):
        assert rel_err(y[0].cpu().numpy(), r[0]) <= TOL, spec


def test_group_gemv_ragged_and_long_groups(q):
    """Ragged K/N (padding panels, partial stages), g = 256 / 512 / 768 / full
    column (one (s, z) group per superstep), 2 tokens, repeat runs identical."""
    specs = [(544, 1000, 4, 32), (288, 40, 3, None), (1024, 17, 2, 64), (768, 300, 4, 256),
             (1536, 520, 3, 512), (2304, 64, 4, 768), (4352, 4000, 2, 128), (96, 24, 4, None)]
    grp, entries, refs = _group_cases(q, specs, seed=11, tokens=2)
    grp.run()
    torch.cuda.synchronize()
    first = [y.clone() for _, _, y in entries]
    for (pw, x, y), r, spec in zip(entries, refs, specs):
        for t in range(2):
            assert rel_err(y[t].cpu().numpy(), r[t]) <= TOL, (spec, t)
    grp.run()
    torch.cuda.synchronize()
    for (_, _, y), f in zip(entries, first):
        assert torch.equal(y, f)  # deterministic


@pytest.mark.parametrize("dtype", [torch.float16, torch.bfloat16])
def test_group_gemv_half_activations(q, dtype):
    specs = [(4096, 1024, 4, 128), (2048, 512, 3, 64), (1024, 2048, 2, 32)]
    grp, entries, refs = _group_cases(q, specs, seed=5, dtype=dtype)
    grp.run()
    torch.cuda.synchronize()
    for (pw, x, y), r, spec in zip(entries, refs, specs):
        assert rel_err(y[0].cpu().numpy(), r[0]) <= TOL_HALF, spec


def test_group_gemv_matches_single_gemv_and_sees_new_inputs(q):
    """Grouped == per-GEMV kernel to f32 rounding; x is referenced, so a
    rewrite of x changes the next run; graph capture works."""
    specs = [(4096, 4096, 4, 128), (11008, 4096, 3, 64)]
    grp, entries, refs = _group_cases(q, specs, seed=21)
    s = torch.cuda.Stream()
    with torch.cuda.stream(s):
        grp.run()
        s.synchronize()
        gph = torch.cuda.CUDAGraph()
        with torch.cuda.graph(gph, stream=s):
            grp.run()
    for pw, x, y in entries:
        x.mul_(-2.0)
    gph.replay()
    torch.cuda.synchronize()
    for pw, x, y in entries:
        ys = pw.gemv(x)
        assert rel_err(y.cpu().numpy(), ys.cpu().numpy()) <= 2e-6


def test_group_gemv_back_to_back_launches_early_trigger(q):
    """Steps issued as plain stream launches, so each prep kernel is a
    programmatic dependent of the previous grouped kernel, with and without the
    prep kernel's early trigger (qigen_debug_group_mode(32)): every step must
    see the previous one complete (records, schedule counter, zeroed split y)."""
    from paper_2307_03738_b200 import _lib
    specs = [(4096, 4096, 4, 128), (11008, 4096, 3, 64), (512, 256, 2, 32), (1024, 64, 4, None)]
    grp, entries, refs = _group_cases(q, specs, seed=31)
    try:
        for mode in (0, 32):
            _lib.lib().qigen_debug_group_mode(mode)
            for _ in range(8):
                grp.run()
            torch.cuda.synchronize()
            for (pw, x, y), r, spec in zip(entries, refs, specs):
                assert rel_err(y[0].cpu().numpy(), r[0]) <= TOL, (mode, spec)
    finally:
        _lib.lib().qigen_debug_group_mode(0)


def test_group_gemv_run_host_c_abi(q):
    """qigen_gemv_group_run_host: pinned host x in, pinned host y out, one call."""
    from paper_2307_03738_b200 import _lib
    from paper_2307_03738_b200.runtime import GemvGroup
    specs = [(1024, 512, 4, 64), (2048, 256, 2, None)]
    rng = np.random.default_rng(41)
    pws = [q.PanelWeights.from_codes(_case(q, K, N, b, g, seed=41 + i)[0])
           for i, (K, N, b, g) in enumerate(specs)]
    koff = np.cumsum([0] + [K for K, *_ in specs])
    noff = np.cumsum([0] + [N for _, N, *_ in specs])
    xd = torch.zeros(int(koff[-1]), device="cuda")
    yd = torch.zeros(int(noff[-1]), device="cuda")
    grp = GemvGroup([(pw, xd[koff[i]:koff[i + 1]], yd[noff[i]:noff[i + 1]])
                     for i, pw in enumerate(pws)])
    xh = torch.from_numpy(rng.normal(0, 1, int(koff[-1])).astype(np.float32)).pin_memory()
    yh = torch.full((int(noff[-1]),), float("nan")).pin_memory()
    _lib.call("qigen_gemv_group_run_host", grp._h, xh.data_ptr(), xd.data_ptr(), xh.numel() * 4,
              yd.data_ptr(), yh.data_ptr(), yh.numel() * 4, torch.cuda.current_stream().cuda_stream)
    for i, pw in enumerate(pws):
        ref = pw.gemv(xh[koff[i]:koff[i + 1]].cuda()).cpu()
        assert rel_err(yh[noff[i]:noff[i + 1]].numpy(), ref.numpy()) <= 2e-6
    with pytest.raises(Exception):
        _lib.call("qigen_gemv_group_run_host", grp._h, None, xd.data_ptr(), 4, yd.data_ptr(),
                  yh.data_ptr(), 4, torch.cuda.current_stream().cuda_stream)


def test_group_gemv_run_rebased(q):
    """qigen_gemv_group_run_rebased: one plan writes to a different output block
    per run (device block and pinned host block); the plan's own y is untouched."""
    from paper_2307_03738_b200 import _lib
    from paper_2307_03738_b200.runtime import GemvGroup
    specs = [(1024, 512, 4, 64), (4096, 4096, 3, 128), (512, 64, 2, None)]
    grp0, entries, refs = _group_cases(q, specs, seed=51)
    noff = np.cumsum([0] + [N for _, N, *_ in specs])
    y0 = torch.full((int(noff[-1]),), float("nan"), device="cuda")
    grp = GemvGroup([(pw, x, y0[noff[i]:noff[i + 1]]) for i, (pw, x, _) in enumerate(entries)])
    st = torch.cuda.current_stream().cuda_stream
    for blk in (torch.zeros(int(noff[-1]), device="cuda"),
                torch.zeros(int(noff[-1])).pin_memory()):
        _lib.call("qigen_gemv_group_run_rebased", grp._h, y0.data_ptr(), blk.data_ptr(), st)
        torch.cuda.synchronize()
        out = blk.cpu().numpy()
        for i, r in enumerate(refs):
            assert rel_err(out[noff[i]:noff[i + 1]], r[0]) <= TOL, (blk.device, specs[i])
    assert torch.isnan(y0).all()


def test_group_gemv_rejects_bad_input(q):
    """The grouped kernel does not take g = 16 (qgemv_batch routes it to single GEMVs)."""
    from paper_2307_03738_b200.runtime import GemvGroup
    cm, *_ = _case(q, 512, 64, 4, 16)
    pw = q.PanelWeights.from_codes(cm)
    with pytest.raises(Exception):
        GemvGroup([(pw, torch.zeros(512, device="cuda"), torch.zeros(64, device="cuda"))])


def test_qgemv_batch_public_api(q):
    """qgemv_batch over reference-format PackedMatrix objects, host in/out."""
    pms, xs, refs = [], [], []
    for i, (K, N, b, g) in enumerate([(1024, 512, 4, 128), (2048, 300, 3, 32), (512, 1024, 2, None)]):
        cm, codes, s, z, rng = _case(q, K, N, b, g, seed=40 + i)
        pms.append(q.lay_out_blocks(cm, q.plan(q.DEFAULT_HARDWARE, cm.config, (K, N))))
        xs.append(rng.normal(0, 1, K).astype(np.float32))
        refs.append(orc.qgemv_reference(codes, s, z, xs[-1]))
    for _ in range(2):  # second call reuses the cached plan
        ys = q.qgemv_batch(pms, xs)
        for y, r in zip(ys, refs):
            assert rel_err(y, r) <= TOL
    # the same list object, mutated in place: the new matrix is used
    cm, codes, s, z, rng = _case(q, 1024, 512, 2, 64, seed=47)
    pms[0] = q.lay_out_blocks(cm, q.plan(q.DEFAULT_HARDWARE, cm.config, (1024, 512)))
    refs[0] = orc.qgemv_reference(codes, s, z, xs[0])
    ys = q.qgemv_batch(pms, xs)
    for y, r in zip(ys, refs):
        assert rel_err(y, r) <= TOL
    # mixed host inputs (a CPU tensor and a float64 array) take the general path
    xs2 = [torch.from_numpy(xs[0]), xs[1].astype(np.float64), xs[2]]
    for y, r in zip(q.qgemv_batch(pms, xs2), refs):
        assert rel_err(y, r) <= TOL
    with pytest.raises(q.ConfigError):
        q.qgemv_batch(pms, [xs[0], xs[1][:-1], xs[2]])


@pytest.mark.parametrize("tokens", [1, 2, 3, 8])
@pytest.mark.parametrize("K,N,bits,g", [(4096, 1536, 4, 128), (2048, 4000, 3, 64), (8192, 512, 2, 32)])
def test_rmsnorm_folded_prologue(q, tokens, K, N, bits, g):
    """prologue "rmsnorm_folded": y = rsqrt(mean(x^2) + eps) (x W) with the
    norm applied in the epilogue from the chunks' sums of squares (rank order)."""
    cm, codes, s, z, rng = _case(q, K, N, bits, g, seed=K + tokens)
    pw = q.PanelWeights.from_codes(cm)
    X = rng.normal(0, 1, (tokens, K)).astype(np.float32) * 3.0
    eps = 1e-5
    Y = pw.gemv(torch.from_numpy(X).cuda(), prologue="rmsnorm_folded", eps=eps).cpu().numpy()
    Y2 = pw.gemv(torch.from_numpy(X).cuda(), prologue="rmsnorm_folded", eps=eps).cpu().numpy()
    assert np.array_equal(Y, Y2)  # deterministic
    for t in range(tokens):
        inv = 1.0 / np.sqrt(np.mean(X[t].astype(np.float64) ** 2) + eps)
        yref = orc.qgemv_reference(codes, s, z, X[t]) * inv
        assert rel_err(Y[t], yref) <= TOL, (tokens, t)


def test_qgemv_batch_device_inputs(q):
    """qgemv_batch with CUDA tensors in and out (no host staging)."""
    pms, xs, refs = [], [], []
    for i, (K, N, b, g) in enumerate([(512, 256, 4, 64), (768, 100, 3, None)]):
        cm, codes, s, z, rng = _case(q, K, N, b, g, seed=60 + i)
        pms.append(q.lay_out_blocks(cm, q.plan(q.DEFAULT_HARDWARE, cm.config, (K, N))))
        x = rng.normal(0, 1, K).astype(np.float32)
        xs.append(torch.from_numpy(x).cuda())
        refs.append(orc.qgemv_reference(codes, s, z, x))
    ys = q.qgemv_batch(pms, xs)
    for y, r in zip(ys, refs):
        assert y.is_cuda and rel_err(y.cpu().numpy(), r) <= TOL


@pytest.mark.parametrize("gc", [32, 64, 128, None])
@pytest.mark.parametrize("tokens", [1, 3])
def test_gemv_chain_digit_epilogue(q, gc, tokens):
    """qigen_gemv_chain: a producer GEMV (residual add) writes its output as the
    consumer's activation digits (times the consumer's RMSNorm weight) plus
    per-CTA sums of squares; the consumer reads the digits and applies 1 / rms
    in its epilogue.  Against the same two steps done separately (RMSNorm in
    torch float64, then the oracle-checked GEMV)."""
    from paper_2307_03738_b200.runtime import digits_buffer, ss_count
    K1, d, M2 = 2048, 1280, 768
    rng = np.random.default_rng(7 + tokens + (gc or 0))
    P = q.PanelWeights.from_float(rng.normal(0, 0.02, (K1, d)).astype(np.float32),
                                  q.QuantConfig(4, 128))
    cmc = q.quantize_matrix(rng.normal(0, 0.02, (d, M2)).astype(np.float32), q.QuantConfig(3, gc))
    C = q.PanelWeights.from_codes(cmc)
    codes, s, z = cmc.numpy()
    x = torch.from_numpy(rng.normal(0, 1, (tokens, K1)).astype(np.float32)).cuda()
    h = torch.from_numpy(rng.normal(0, 1, (tokens, d)).astype(np.float32)).cuda()
    w = torch.from_numpy(rng.uniform(0.5, 1.5, d).astype(np.float32)).cuda()
    h_ref = h + P.gemv(x)
    dig = digits_buffer(d, tokens, "cuda")
    ssc = ss_count(d)
    ss = torch.zeros(tokens * ssc, device="cuda")
    for _ in range(2):  # buffers are reusable
        hh = h.clone()
        P.chain(x, hh, tokens=tokens, accumulate=True, digits_out=dig, out_scale=w, out_group=gc,
                ss_out=ss)
        y = torch.empty(tokens, M2, device="cuda")
        C.chain(None, y, tokens=tokens, digits_in=dig, ss_in=ss, ss_count=ssc, eps=1e-5)
        torch.cuda.synchronize()
        assert torch.allclose(hh, h_ref, rtol=0, atol=1e-5)
        hd = hh.double().cpu().numpy()
        xn = hd / np.sqrt((hd ** 2).mean(-1, keepdims=True) + 1e-5) * w.double().cpu().numpy()
        ref = orc.qgemv_reference(codes, s, z, xn)
        assert rel_err(y.cpu().numpy(), ref) <= TOL, (gc, tokens, rel_err(y.cpu().numpy(), ref))
        assert np.allclose(ss.view(tokens, ssc).sum(1).cpu().numpy(), (hd ** 2).sum(1), rtol=1e-5)


@pytest.mark.gpu
def test_qgemv_batch_pinned_inputs(q):
    """qgemv_batch_inputs: numpy views of the pinned gather buffer, filled in
    place, are read by the grouped launch without a host gather; fresh inputs on
    every call give that call's results, earlier results stay intact, and a
    list of other arrays still takes the gathering path."""
    rng = np.random.default_rng(5)
    pms, cms = [], []
    for (K, N, b, g) in [(1024, 768, 4, 128), (2048, 512, 3, 64), (512, 1040, 2, 32)]:
        w = rng.normal(0, 0.02, (K, N)).astype(np.float32)
        cm = q.quantize_matrix(w, q.QuantConfig(b, g))
        cms.append(cm)
        pms.append(q.lay_out_blocks(cm, q.plan(q.DEFAULT_HARDWARE, cm.config, (K, N))))
    xs_pin = q.qgemv_batch_inputs(pms)
    assert [x.shape for x in xs_pin] == [(pm.n,) for pm in pms]
    kept = []
    for rep in range(3):
        xs = [rng.normal(0, 1, pm.n).astype(np.float32) for pm in pms]
        for dst, src in zip(xs_pin, xs):
            np.copyto(dst, src)
        ys = q.qgemv_batch(pms, xs_pin)
        refs = [orc.qgemv_reference(*cm.numpy(), x) for cm, x in zip(cms, xs)]
        for y, r in zip(ys, refs):
            assert np.abs(y - r).max() / (1 + np.abs(r).max()) <= 1e-5
        kept.append((ys, refs))
    for ys, refs in kept:  # earlier calls' result blocks were not overwritten
        for y, r in zip(ys, refs):
            assert np.abs(y - r).max() / (1 + np.abs(r).max()) <= 1e-5
    xs = [rng.normal(0, 1, pm.n).astype(np.float32) for pm in pms]
    ys = q.qgemv_batch(pms, xs)  # plain arrays: gathered
    for y, cm, x in zip(ys, cms, xs):
        r = orc.qgemv_reference(*cm.numpy(), x)
        assert np.abs(y - r).max() / (1 + np.abs(r).max()) <= 1e-5
