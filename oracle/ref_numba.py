"""The REFERENCE's own CPU qGEMV, run as shipped — TEST / BASELINE INFRASTRUCTURE ONLY.

Used by ``bench.py``'s ``--impl reference`` arm and ``cpu_baseline`` leg (and by
nothing in ``paper_2307_03738_b200/``).  It imports the unmodified reference
package ``qigen`` — from ``baseline/_ref`` (installed there once with
``pip install --no-index --no-build-isolation --no-deps --target baseline/_ref``
from a copy of ``/root/reference/pkg``; git-ignored, travels to the GPU box) or
from ``/root/reference/pkg/src`` in the build container — and runs its
generated qGEMV kernel (``kernelgen.generate_qgemv``, kernelgen.py:371-423)
JIT-compiled by numba through the reference's own ``vecops.jit_kernel``
(vecops.py:103-105), i.e. BASELINE.md §2's "reference's own optimized CPU path".

The reference ships no runtime and its generator needs two
documented import-time shims (the same ones
``tests/golden/make_golden.py`` applies, without editing the reference):
  * F3: ``_WordAccess`` is called without ``k_words`` (kernelgen.py:201, :351);
  * F4: full-column kernels index x by word group instead of row
    (kernelgen.py:254-257); fixed in the generated source text.
The runtime is reconstructed per SURVEY Appendix B (exec layout from
``qigen_oracle.ExecLayout``; T threads own disjoint column-block ranges,
SPEC.md:376).
"""

from __future__ import annotations

import sys
import threading
from pathlib import Path

import numpy as np

ROOT = Path(__file__).resolve().parents[1]
_CANDIDATES = [ROOT / "baseline" / "_ref", Path("/root/reference/pkg/src")]
_MOD = None


def available() -> str | None:
    """Path the reference imports from, or None if it is not present here."""
    for p in _CANDIDATES:
        if (p / "qigen" / "kernelgen.py").exists():
            return str(p)
    return None


def _load():
    global _MOD
    if _MOD is not None:
        return _MOD
    path = available()
    if path is None:
        raise ImportError("the reference package (baseline/_ref) is not installed")
    if path not in sys.path:
        sys.path.insert(0, path)
    from qigen import config as qcfg
    from qigen import kernelgen, perfmodel, vecops
    from qigen.config import QuantConfig

    cur_kw = [1]
    orig = kernelgen._WordAccess

    class _WordAccessShim(orig):  # F3
        def __init__(self, cached, t_b, lanes, k_words=None, fragment=False):
            super().__init__(cached, t_b, lanes, cur_kw[0] if k_words is None else k_words,
                             fragment)

    kernelgen._WordAccess = _WordAccessShim

    def load_kernel(bits, g, tp):
        desc = kernelgen.KernelDescriptor(bits, g, tp)
        unit, kw = qcfg.pack_unit(bits)
        cur_kw[0] = kw
        text = kernelgen.generate_qgemv(desc).source_text
        if g is None:  # F4
            text = text.replace("px = xbase + wg", f"px = xbase // {unit} + wg")
        ns: dict = {}
        exec(compile(text, desc.filename, "exec"), ns)
        return vecops.jit_kernel(ns[desc.name])

    _MOD = dict(load_kernel=load_kernel, perfmodel=perfmodel, QuantConfig=QuantConfig)
    return _MOD


class RefKernel:
    """The reference's numba kernel for one matrix (exec layout + compiled
    kernel), callable with T threads like the reference runtime."""

    def __init__(self, ex, bits: int, g, plan):
        m = _load()
        self.ex, self.bits, self.g = ex, bits, g
        self.kern = m["load_kernel"](bits, g, m["perfmodel"].TilePlan(*plan))
        self.s = ex.scales.reshape(-1)
        self.z = ex.zeros.reshape(-1)
        self._parts = {}

    def _partition(self, threads):
        """Per thread: its column-block range and block descriptors."""
        if threads not in self._parts:
            ex, cbs = self.ex, self.ex.cbs
            cuts = [cbs * i // threads for i in range(threads + 1)]
            parts = []
            for i in range(threads):
                lo, hi = cuts[i], cuts[i + 1]
                if hi <= lo:
                    continue
                sel = (ex.blk_cb >= lo) & (ex.blk_cb < hi)
                parts.append((lo, hi, np.ascontiguousarray(ex.blk_off[sel]),
                              np.ascontiguousarray(ex.blk_rb[sel]),
                              np.ascontiguousarray(ex.blk_cb[sel]), int(sel.sum())))
            self._parts[threads] = parts
        return self._parts[threads]

    def __call__(self, x: np.ndarray, threads: int = 1) -> np.ndarray:
        ex = self.ex
        xp = ex.pad_x(x)
        xs = ex.xsums(xp)
        y = np.zeros(ex.m_pad, dtype=np.float32)
        cbs = ex.cbs

        def run(part):
            lo, hi, off, rb, cb, nb = part
            self.kern(ex.words, self.s, self.z, xp, xs, y, ex.n, ex.m, off, rb, cb, nb, lo, hi,
                      cbs)

        parts = self._partition(max(1, threads))
        if len(parts) == 1:
            run(parts[0])
        else:
            ths = [threading.Thread(target=run, args=(p,)) for p in parts]
            for t in ths:
                t.start()
            for t in ths:
                t.join()
        return y[: ex.m].copy()
