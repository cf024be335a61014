"""Generate the golden fixtures by running the REFERENCE implementation.

Run in the build container (where /root/reference exists):

    NUMBA_DISABLE_JIT=1 python tests/golden/make_golden.py

It imports qigen from /root/reference/pkg/src (read-only, never copied), applies
the two import-time shims SURVEY.md §8(c) documents (F3: pass ``k_words`` to
``_WordAccess``; F4: fix the full-column x index in generated source text), and
writes small .npz/.json fixtures next to this file.  The fixtures travel with the
repo; the GPU box never needs /root/reference.

Fixtures:
  quant_pack.npz  — reference quantize_matrix outputs (codes/scales/zeros with
                    signed zeros) and ROW_SEQUENTIAL + ZCURVE packed words.
  plans.json      — reference perfmodel.plan() results.
  qgemv.npz       — outputs of the reference's generated qGEMV kernels (executed
                    by the reference's own vecops layer) on the exec layout of
                    SURVEY Appendix B, with the x / xsums they were fed.
  kats.json       — the SPEC examples evaluated by the reference code.
"""

from __future__ import annotations

import json
import os
import sys
from pathlib import Path

import numpy as np

REF = "/root/reference/pkg/src"
HERE = Path(__file__).resolve().parent
sys.path.insert(0, REF)
sys.path.insert(0, str(HERE.parents[1]))

from qigen import config as qcfg  # noqa: E402
from qigen import kernelgen, packing, perfmodel, quant, vecops  # noqa: E402
from qigen.config import QuantConfig, ZeroMode  # noqa: E402

from oracle import qigen_oracle as orc  # noqa: E402  (exec-layout builder only)

# --- shim F3 (kernelgen.py:201, :351 call _WordAccess without k_words) -------
_CUR_KW = [1]
_OrigWA = kernelgen._WordAccess


class _WordAccessShim(_OrigWA):
    def __init__(self, cached, t_b, lanes, k_words=None, fragment=False):
        super().__init__(cached, t_b, lanes, _CUR_KW[0] if k_words is None else k_words,
                         fragment)


kernelgen._WordAccess = _WordAccessShim


def generate_source(desc: kernelgen.KernelDescriptor) -> str:
    unit, kw = qcfg.pack_unit(desc.bits)
    _CUR_KW[0] = kw
    text = kernelgen.generate_qgemv(desc).source_text
    if desc.group_size is None:  # shim F4 (kernelgen.py:254-257)
        assert "px = xbase + wg" in text
        text = text.replace("px = xbase + wg", f"px = xbase // {unit} + wg")
    return text


def load_kernel(desc):
    ns: dict = {}
    exec(compile(generate_source(desc), desc.filename, "exec"), ns)
    return vecops.jit_kernel(ns[desc.name])


def main() -> None:
    rng = np.random.default_rng(20230707)
    out_qp: dict[str, np.ndarray] = {}
    cases = []
    shapes = [(64, 48), (192, 40), (96, 56)]
    groups = [16, 32, 64, None]
    ci = 0
    for bits in (2, 3, 4):
        for (n, m) in shapes:
            if n % qcfg.pack_unit(bits)[0]:
                continue
            for g in groups:
                if g is not None and n % g:
                    continue
                for zm in ("real32", "quantized"):
                    w = rng.normal(0.0, 0.02, (n, m)).astype(np.float32)
                    # special columns: constant, all-zero (-0.0 z), exact ties, -0.0 entries
                    w[:, 0] = 0.37
                    w[:, 1] = 0.0
                    if m > 3:
                        w[:, 2] = np.tile(np.array([0.0, 0.5, 3.0, 1.5], np.float32), n // 4)
                        w[: n // 2, 3] = -0.0
                    if m > 5:  # min is a signed zero: the last of +0/-0 decides z's sign
                        w[:, 4] = np.abs(w[:, 4])
                        w[::5, 4] = 0.0
                        w[::7, 4] = -0.0
                        w[:, 5] = -np.abs(w[:, 5])
                        w[1::3, 5] = -0.0
                        w[2::5, 5] = 0.0
                    cm = quant.quantize_matrix(w, QuantConfig(bits, g, zm))
                    unit = qcfg.pack_unit(bits)[0]
                    m_b = 3 * (unit if g is None else int(np.lcm(unit, g)))
                    m_b = m_b * max(1, (n // 3) // m_b)  # several (ragged) row blocks
                    t_b = 24 * max(1, (m // 2) // 24)
                    tp = perfmodel.TilePlan(3, 3, m_b, t_b)
                    pz = packing.lay_out_blocks(cm, tp, packing.Layout.ZCURVE)
                    pr = packing.lay_out_blocks(cm, tp, packing.Layout.ROW_SEQUENTIAL)
                    key = f"c{ci}"
                    out_qp[key + "_w"] = w
                    out_qp[key + "_codes"] = cm.codes
                    out_qp[key + "_scales"] = cm.scales
                    out_qp[key + "_zeros"] = cm.zeros
                    out_qp[key + "_rowseq"] = pr.words
                    out_qp[key + "_zcurve"] = pz.words
                    cases.append(dict(key=key, bits=bits, n=n, m=m, g=g, zero_mode=zm,
                                      m_b=m_b, t_b=t_b))
                    ci += 1
    np.savez_compressed(HERE / "quant_pack.npz", **out_qp)
    (HERE / "quant_pack.json").write_text(json.dumps(cases, indent=1))

    # --- plans ---------------------------------------------------------------
    plans = []
    dims_list = [(4096, 4096), (4096, 11008), (11008, 4096), (8192, 8192), (8192, 22016),
                 (22016, 8192), (64, 64), (96, 48), (1024, 1024), (32, 24), (5504, 4096)]
    for bits in (2, 3, 4):
        for g in (16, 32, 64, 128, None):
            for dims in dims_list:
                unit = qcfg.pack_unit(bits)[0]
                if dims[0] % unit or (g is not None and dims[0] % g):
                    continue
                try:
                    p = perfmodel.plan(perfmodel.DEFAULT_HARDWARE, QuantConfig(bits, g), dims)
                    plans.append(dict(bits=bits, g=g, dims=list(dims),
                                      plan=[p.m_u, p.t_u, p.m_b, p.t_b]))
                except Exception as e:  # noqa: BLE001
                    plans.append(dict(bits=bits, g=g, dims=list(dims), error=type(e).__name__))
    for l1 in (4096, 8192, 65536):
        for vregs in (3, 8, 16, 32):
            for bits in (2, 3, 4):
                hw = perfmodel.HardwareSpec(l1_bits=l1, vregs=vregs)
                try:
                    p = perfmodel.plan(hw, QuantConfig(bits, 32), (256, 512))
                    plans.append(dict(bits=bits, g=32, dims=[256, 512], l1_bits=l1,
                                      vregs=vregs, plan=[p.m_u, p.t_u, p.m_b, p.t_b]))
                except Exception as e:  # noqa: BLE001
                    plans.append(dict(bits=bits, g=32, dims=[256, 512], l1_bits=l1,
                                      vregs=vregs, error=type(e).__name__))
    (HERE / "plans.json").write_text(json.dumps(plans, indent=1))

    # --- qgemv: the reference's generated kernels ------------------------------
    out_q: dict[str, np.ndarray] = {}
    qcases = []
    qi = 0
    for bits in (2, 3, 4):
        unit = qcfg.pack_unit(bits)[0]
        for g in (16, 32, 64, 128, None):
            for (n, m) in [(256, 72), (384, 48), (768, 24)]:
                if n % unit or (g is not None and n % g):
                    continue
                w = rng.normal(0.0, 0.02, (n, m)).astype(np.float32)
                cm = quant.quantize_matrix(w, QuantConfig(bits, g))
                m_align = unit if g is None else int(np.lcm(unit, g))
                # m_b must be a multiple of m_u=3 and the alignment; ragged grids on
                # purpose (several row blocks, last one partial; (256,72) has 48+24 cols)
                step = 3 * m_align
                m_b = step * max(1, (n // 2) // step)
                t_b = 48 if n == 256 else 24
                tp = perfmodel.TilePlan(3, 3, m_b, t_b)
                pr = packing.lay_out_blocks(cm, tp, packing.Layout.ROW_SEQUENTIAL)
                ex = orc.ExecLayout(pr.words, cm.scales, cm.zeros, n, m, bits, g, m_b, t_b)
                x = rng.normal(0.0, 1.0, n).astype(np.float32)
                xp = ex.pad_x(x)
                xs = ex.xsums(xp)
                y = np.zeros(ex.m_pad, dtype=np.float32)
                kern = load_kernel(kernelgen.KernelDescriptor(bits, g, tp))
                kern(ex.words, ex.scales.reshape(-1), ex.zeros.reshape(-1), xp, xs, y, n, m,
                     ex.blk_off, ex.blk_rb, ex.blk_cb, len(ex.blk_off), 0, ex.cbs, ex.cbs)
                key = f"q{qi}"
                out_q[key + "_w"] = w
                out_q[key + "_x"] = x
                out_q[key + "_xsums"] = xs
                out_q[key + "_y"] = y[:m].copy()
                qcases.append(dict(key=key, bits=bits, g=g, n=n, m=m, m_b=m_b, t_b=t_b))
                qi += 1
                print("qgemv golden", key, bits, g, n, m, flush=True)
    np.savez_compressed(HERE / "qgemv.npz", **out_q)
    (HERE / "qgemv.json").write_text(json.dumps(qcases, indent=1))

    # --- KATs (SPEC examples, evaluated by the reference) ----------------------
    kats = {}
    c, p = quant.quantize_group(np.arange(16, dtype=np.float32), 4)
    kats["q_0_15"] = dict(codes=c.tolist(), s=p.scale, z=p.zero, z_signbit=bool(np.signbit(p.zero)))
    c, p = quant.quantize_group(np.full(8, 0.37, np.float32), 4)
    kats["q_const"] = dict(codes=c.tolist(), s=p.scale, z=p.zero)
    c, p = quant.quantize_group(np.array([-1, 1], np.float32), 2)
    kats["q_pm1_b2"] = dict(codes=c.tolist(), s=p.scale, z=p.zero)
    c, p = quant.quantize_group(np.array([-1, 1], np.float32), 2, "quantized")
    kats["q_pm1_b2_quant"] = dict(codes=c.tolist(), s=p.scale, z=p.zero)
    c, p = quant.quantize_group(np.full(4, 0.37, np.float32), 4, "quantized")
    kats["q_const_quant"] = dict(codes=c.tolist(), s=p.scale, z=p.zero,
                                 z_signbit=bool(np.signbit(p.zero)))
    c, p = quant.quantize_group(np.array([0, 0.5, 3], np.float32), 2)
    kats["q_tie_b2"] = dict(codes=c.tolist(), s=p.scale, z=p.zero)
    kats["pack_4"] = int(packing.pack_words(np.arange(1, 9), 4)[0])
    kats["pack_3_all7"] = [int(v) for v in packing.pack_words(np.full(32, 7), 3)]
    kats["pack_3_one"] = [int(v) for v in packing.pack_words(np.array([1] + [0] * 31), 3)]
    kats["pack_2"] = int(packing.pack_words(np.tile(np.arange(4), 4), 2)[0])
    kats["morton"] = {f"{r},{c}": packing.morton_index(r, c)
                      for r, c in [(0, 0), (1, 0), (0, 1), (3, 5), (7, 7), (12, 3)]}
    kats["block_order_2x2"] = [list(t) for t in packing.block_order(2, 2)]
    kats["reg_tile_16"] = list(perfmodel.select_register_tile(perfmodel.HardwareSpec(vregs=16)))
    kats["reg_tile_3"] = list(perfmodel.select_register_tile(perfmodel.HardwareSpec(vregs=3)))
    cm = quant.quantize_matrix(np.zeros((4096, 4096), np.float32)[:, :8], QuantConfig(4, None))
    pm = packing.PackedMatrix(np.zeros(4096 * 4096 // 8, np.uint32), 4096, 4096,
                              QuantConfig(4, None, "quantized"),
                              np.ones((1, 4096), np.float32), np.zeros((1, 4096), np.float32),
                              perfmodel.TilePlan(3, 3, 24, 2040))
    kats["payload_bits_4096_b4_fc_q"] = list(pm.payload_bits())
    del cm
    (HERE / "kats.json").write_text(json.dumps(kats, indent=1))
    print("wrote", sorted(p.name for p in HERE.iterdir()))


if __name__ == "__main__":
    if os.environ.get("NUMBA_DISABLE_JIT") != "1":
        print("note: run with NUMBA_DISABLE_JIT=1 so the generated kernels run interpreted")
    main()
