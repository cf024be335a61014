"""The drop-in boundary: the reference-side binding documented in
INTEGRATION.md, executed verbatim against libqigen_b200.so, and the C ABI's
re-entrancy across streams and host threads (§8(b) "Threading": stream-ordered,
re-entrant, deterministic)."""

import ctypes
import re
import sys
import threading
import types
from pathlib import Path
from types import SimpleNamespace

import numpy as np
import pytest
import torch

from oracle import qigen_oracle as orc

ROOT = Path(__file__).resolve().parents[1]
TOL = 1e-5


def rel_err(y, yref):
    y, yref = np.asarray(y, np.float64), np.asarray(yref, np.float64)
    return np.abs(y - yref).max() / (1.0 + np.abs(yref).max())


def _integration_blocks():
    text = (ROOT / "INTEGRATION.md").read_text()
    return re.findall(r"```python\n(.*?)```", text, flags=re.S)


def test_integration_binding_is_documented():
    """CPU: INTEGRATION.md carries the binding, and it binds exactly the entry
    points the header declares."""
    blocks = _integration_blocks()
    assert len(blocks) >= 2
    header = (ROOT / "include" / "qigen_b200.h").read_text()
    for name in set(re.findall(r"_lib\.(qigen_\w+)", "\n".join(blocks))):
        assert re.search(rf"\b{name}\s*\(", header), name


def _binding_module():
    """Execute INTEGRATION.md's `qigen/runtime_b200.py` verbatim inside a stand-in
    package whose config / packing / perfmodel modules are this repo's mirrors
    of the reference's (same names, same exception classes)."""
    import paper_2307_03738_b200 as q
    from paper_2307_03738_b200 import config, packing, perfmodel
    q._lib.lib()  # loads libqigen_b200.so (soname libqigen_b200.so) by path
    pkg = types.ModuleType("qigen_ref")
    pkg.__path__ = []
    sys.modules["qigen_ref"] = pkg
    for name, mod in (("config", config), ("packing", packing), ("perfmodel", perfmodel)):
        sys.modules[f"qigen_ref.{name}"] = mod
    mod = types.ModuleType("qigen_ref.runtime_b200")
    mod.__package__ = "qigen_ref"
    blocks = _integration_blocks()
    exec(compile(blocks[0] + "\n" + blocks[1], "INTEGRATION.md", "exec"), mod.__dict__)
    return mod


def _reference_packed(q, K, N, bits, g, layout, seed):
    """A reference-style PackedMatrix: numpy words from the oracle's restatement
    of packing.py, numpy scales/zeros, the reference's default plan."""
    rng = np.random.default_rng(seed)
    w = rng.normal(0, 0.02, (K, N)).astype(np.float32)
    codes, s, z = orc.quantize_matrix(w, bits, g)
    cfg = q.QuantConfig(bits, g)
    p = q.plan(q.DEFAULT_HARDWARE, cfg, (K, N))
    words = orc.lay_out_words(codes, bits, p.m_b, p.t_b, layout is q.Layout.ZCURVE)
    pm = SimpleNamespace(words=words, n=K, m=N, config=cfg, scales=s, zeros=z, plan=p,
                         layout=layout, _exec_cache=None)
    return pm, codes, s, z, rng


@pytest.mark.gpu
@pytest.mark.parametrize("layout", ["ROW_SEQUENTIAL", "ZCURVE"])
@pytest.mark.parametrize("K,N,bits,g", [(4096, 4096, 4, 128), (1024, 520, 3, 64),
                                        (2048, 300, 2, None), (768, 1000, 3, 32)])
def test_integration_binding_verbatim(layout, K, N, bits, g):
    """INTEGRATION.md's qgemv: qigen_weights_create (ZCURVE with blk_rc) then
    qigen_weights_gemv_host, against the dense fp64 oracle; the handle is cached
    in pm._exec_cache and reused."""
    import paper_2307_03738_b200 as q
    rt = _binding_module()
    pm, codes, s, z, rng = _reference_packed(q, K, N, bits, g, q.Layout[layout], K + N + bits)
    for _ in range(2):
        x = rng.normal(0, 1, K).astype(np.float32)
        y = rt.qgemv(pm, x)
        assert y.shape == (N,) and y.dtype == np.float32
        assert rel_err(y, orc.qgemv_reference(codes, s, z, x)) <= TOL
    assert pm._exec_cache is not None
    rt._lib.qigen_weights_destroy(pm._exec_cache)


@pytest.mark.gpu
def test_integration_binding_errors():
    """Status codes surface as the reference's exception classes."""
    import paper_2307_03738_b200 as q
    rt = _binding_module()
    pm, *_ = _reference_packed(q, 512, 64, 4, 64, q.Layout.ROW_SEQUENTIAL, 1)
    pm.config = SimpleNamespace(bits=5, group_size=64)  # invalid bit width
    with pytest.raises(q.ConfigError):
        rt.qgemv(pm, np.zeros(512, np.float32))


@pytest.mark.gpu
def test_integration_group_binding():
    """INTEGRATION.md's make_group over device panels, run on a stream."""
    import paper_2307_03738_b200 as q
    rt = _binding_module()
    specs = [(1024, 512, 4, 64), (768, 200, 3, None)]
    panels, keep, refs = [], [], []
    for i, (K, N, b, g) in enumerate(specs):
        rng = np.random.default_rng(70 + i)
        w = rng.normal(0, 0.02, (K, N)).astype(np.float32)
        pw = q.PanelWeights.from_float(w, q.QuantConfig(b, g))
        codes, s, z = orc.quantize_matrix(w, b, g)
        x = rng.normal(0, 1, K).astype(np.float32)
        xd, yd = torch.from_numpy(x).cuda(), torch.full((N,), float("nan"), device="cuda")
        panels.append((pw.qw.data_ptr(), pw.qsz.data_ptr(), K, N, b, g or 0, xd.data_ptr(),
                       yd.data_ptr()))
        keep += [pw, xd, yd]
        refs.append((yd, orc.qgemv_reference(codes, s, z, x)))
    h = rt.make_group(panels)
    rt._check(rt._lib.qigen_gemv_group_run(h, ctypes.c_void_p(torch.cuda.current_stream().cuda_stream)))
    torch.cuda.synchronize()
    for yd, ref in refs:
        assert rel_err(yd.cpu().numpy(), ref) <= TOL
    rt._lib.qigen_gemv_group_destroy(h)


# --- re-entrancy across streams and threads ---------------------------------------

@pytest.mark.gpu
def test_gemv_reentrant_across_streams():
    """qigen_gemv without a caller workspace (the library's stream-ordered
    scratch) on two streams at once, many times: every result bit-identical to
    the serial one.  Shapes force the activation prep kernel (long K chunks)."""
    import paper_2307_03738_b200 as q
    from paper_2307_03738_b200 import _lib
    L = _lib.lib()
    K, N, T = 11008, 512, 8
    rng = np.random.default_rng(3)
    pw = q.PanelWeights.from_float(rng.normal(0, 0.02, (K, N)).astype(np.float32),
                                   q.QuantConfig(4, 128))
    xs = [torch.from_numpy(rng.normal(0, 1, (T, K)).astype(np.float32)).cuda() for _ in range(2)]
    ref = [pw.gemv(x) for x in xs]
    torch.cuda.synchronize()
    streams = [torch.cuda.Stream() for _ in range(2)]
    outs = [[torch.empty(T, N, device="cuda") for _ in range(20)] for _ in range(2)]
    for i in range(20):
        for j in range(2):
            _lib.call("qigen_gemv", pw.qw.data_ptr(), pw.qsz.data_ptr(), K, N, 4, 128,
                      xs[j].data_ptr(), 0, T, K, outs[j][i].data_ptr(), N, 0, 0,
                      streams[j].cuda_stream)
    torch.cuda.synchronize()
    for j in range(2):
        for o in outs[j]:
            assert torch.equal(o, ref[j])
    assert L is not None


@pytest.mark.gpu
def test_weights_handle_from_threads():
    """One qigen_weights handle, blocking host-buffer calls from 4 host threads on
    their own streams: every result equals the single-threaded one."""
    import paper_2307_03738_b200 as q
    from paper_2307_03738_b200 import _lib
    K, N, bits, g = 4096, 1024, 3, 64
    rng = np.random.default_rng(5)
    w = rng.normal(0, 0.02, (K, N)).astype(np.float32)
    cm = q.quantize_matrix(w, q.QuantConfig(bits, g))
    pm = q.lay_out_blocks(cm, q.plan(q.DEFAULT_HARDWARE, cm.config, (K, N)),
                          q.Layout.ROW_SEQUENTIAL)
    h = ctypes.c_void_p()
    _lib.call("qigen_weights_create", pm.words.data_ptr(), 0, K, N, bits, g, 0, 0, None, 0,
              cm.scales.data_ptr(), cm.zeros.data_ptr(), None, ctypes.byref(h))
    xs = [rng.normal(0, 1, (2, K)).astype(np.float32) for _ in range(4)]
    expect = []
    for x in xs:
        y = np.empty((2, N), np.float32)
        _lib.call("qigen_weights_gemv_host", h, x.ctypes.data, 2, y.ctypes.data, None)
        expect.append(y)
    errors = []

    def worker(i):
        try:
            torch.cuda.set_device(0)
            s = torch.cuda.Stream()
            for _ in range(25):
                y = np.empty((2, N), np.float32)
                _lib.call("qigen_weights_gemv_host", h, xs[i].ctypes.data, 2, y.ctypes.data,
                          ctypes.c_void_p(s.cuda_stream))
                if not np.array_equal(y, expect[i]):
                    errors.append(i)
        except Exception as e:  # noqa: BLE001
            errors.append(repr(e))

    ths = [threading.Thread(target=worker, args=(i,)) for i in range(4)]
    for t in ths:
        t.start()
    for t in ths:
        t.join()
    _lib.lib().qigen_weights_destroy(h)
    assert not errors, errors
    codes, s_, z_ = cm.numpy()
    assert rel_err(expect[0][1], orc.qgemv_reference(codes, s_, z_, xs[0][1])) <= TOL


@pytest.mark.gpu
def test_qgemv_batch_threads_and_fresh_inputs():
    """qgemv_batch on one cached matrix list: fresh activations every call (each
    result checked against its own reference, earlier results kept and
    re-checked: distinct output blocks), then 3 threads calling concurrently."""
    import paper_2307_03738_b200 as q
    pms, mats = [], []
    for i, (K, N, b, g) in enumerate([(1024, 512, 4, 128), (2048, 300, 3, 32), (512, 1024, 2, None)]):
        rng = np.random.default_rng(80 + i)
        w = rng.normal(0, 0.02, (K, N)).astype(np.float32)
        cm = q.quantize_matrix(w, q.QuantConfig(b, g))
        pms.append(q.lay_out_blocks(cm, q.plan(q.DEFAULT_HARDWARE, cm.config, (K, N))))
        mats.append(orc.dequantize_matrix(*cm.numpy()).astype(np.float64))
    rng = np.random.default_rng(9)
    kept = []
    for _ in range(6):
        xs = [rng.normal(0, 1, m.shape[0]).astype(np.float32) for m in mats]
        ys = q.qgemv_batch(pms, xs)
        kept.append((xs, ys))
        for x, y, m in zip(xs, ys, mats):
            assert rel_err(y, x.astype(np.float64) @ m) <= TOL
    for xs, ys in kept:  # earlier results are still their own
        for x, y, m in zip(xs, ys, mats):
            assert rel_err(y, x.astype(np.float64) @ m) <= TOL
    errors = []

    def worker(seed):
        try:
            torch.cuda.set_device(0)
            r = np.random.default_rng(seed)
            for _ in range(15):
                xs = [r.normal(0, 1, m.shape[0]).astype(np.float32) for m in mats]
                for x, y, m in zip(xs, q.qgemv_batch(pms, xs), mats):
                    if rel_err(y, x.astype(np.float64) @ m) > TOL:
                        errors.append(seed)
        except Exception as e:  # noqa: BLE001
            errors.append(repr(e))

    ths = [threading.Thread(target=worker, args=(s,)) for s in range(3)]
    for t in ths:
        t.start()
    for t in ths:
        t.join()
    assert not errors, errors


@pytest.mark.gpu
def test_group_rejects_unaddressable_outputs():
    """Pageable host y is rejected at create (GemvGroup and the C ABI); a plan
    with device y whose GEMVs are K-split cannot be rebased onto host memory."""
    import paper_2307_03738_b200 as q
    from paper_2307_03738_b200 import _lib
    from paper_2307_03738_b200.runtime import GemvGroup
    rng = np.random.default_rng(2)
    big = q.PanelWeights.from_float(rng.normal(0, 0.02, (8192, 4096)).astype(np.float32),
                                    q.QuantConfig(4, 128))
    small = q.PanelWeights.from_float(rng.normal(0, 0.02, (2048, 256)).astype(np.float32),
                                      q.QuantConfig(2, 64))
    xb, xs_ = torch.randn(8192, device="cuda"), torch.randn(2048, device="cuda")
    with pytest.raises(q.ConfigError):
        GemvGroup([(small, xs_, torch.zeros(256))])  # pageable CPU y
    y0 = torch.zeros(4096 + 256, device="cuda")
    grp = GemvGroup([(big, xb, y0[:4096]), (small, xs_, y0[4096:])])
    grp.run()
    torch.cuda.synchronize()
    ref = torch.cat([big.gemv(xb), small.gemv(xs_)])
    assert ((y0 - ref).abs().max() / (1 + ref.abs().max())).item() <= 2e-6
    st = torch.cuda.current_stream().cuda_stream
    host = torch.zeros(y0.numel()).pin_memory()
    # the small GEMV costs < 20 % of the big one: it is K-split (atomics into y)
    with pytest.raises(ValueError):
        _lib.call("qigen_gemv_group_run_rebased", grp._h, y0.data_ptr(), host.data_ptr(), st)
    pageable = np.zeros(y0.numel(), np.float32)
    with pytest.raises(ValueError):
        _lib.call("qigen_gemv_group_run_rebased", grp._h, y0.data_ptr(), pageable.ctypes.data, st)
    dev2 = torch.zeros_like(y0)
    _lib.call("qigen_gemv_group_run_rebased", grp._h, y0.data_ptr(), dev2.data_ptr(), st)
    torch.cuda.synchronize()
    assert ((dev2 - ref).abs().max() / (1 + ref.abs().max())).item() <= 2e-6
