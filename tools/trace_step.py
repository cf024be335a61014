"""Timeline of the real decode step (LlamaTP.step, chained or not): per GEMV /
attention launch of the last traced layers, CTA entry, PDL wait, prologue done,
main loop done, exit (globaltimer, us from the step's first CTA entry).
  python tools/trace_step.py [7b|65b] [layers] [batch]"""
import math
import sys
from pathlib import Path

import numpy as np
import torch

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
from paper_2307_03738_b200 import _lib, decode as D  # noqa: E402

name = sys.argv[1] if len(sys.argv) > 1 else "7b"
L = int(sys.argv[2]) if len(sys.argv) > 2 else 4
B = int(sys.argv[3]) if len(sys.argv) > 3 else 1
base, ctx = (D.LLAMA_7B, 512) if name == "7b" else (D.LLAMA_65B, 1024)
cfg = D.shrink(base, n_layers=L)
m = D.LlamaTP(cfg, batch=B, max_ctx=ctx + 1, seed=0)
Lb = _lib.lib()
bufs, order = {}, []
state = {"i": 0}
names = ["qkv", "o", "gu", "down"]


def buf(key, n=16):
    if key not in bufs:
        bufs[key] = torch.zeros(8192 * n, dtype=torch.int64, device="cuda")
        order.append(key)
    return bufs[key]


def wrap(meth):
    def f(self, *a, **k):
        key = (state["i"] // 4, names[state["i"] % 4])
        state["i"] += 1
        Lb.qigen_debug_trace(buf(key).data_ptr())
        try:
            return meth(self, *a, **k)
        finally:
            Lb.qigen_debug_trace(None)
    return f


D.GpuLinear.__call__ = wrap(D.GpuLinear.__call__)
D.GpuLinear.chain = wrap(D.GpuLinear.chain)
att0 = D.GpuBackend.attention


def attn(*a, **kw):
    key = (state["i"] // 4, "attn")
    Lb.qigen_debug_attn_trace(buf(key, 4).data_ptr())
    try:
        att0(*a, **kw)
    finally:
        Lb.qigen_debug_attn_trace(None)


D.GpuBackend.attention = staticmethod(attn)
tok = torch.zeros(B, dtype=torch.long, device="cuda")
s = torch.cuda.Stream()
with torch.cuda.stream(s):
    state["i"] = 0
    m.step(tok, ctx)
    s.synchronize()
    g = torch.cuda.CUDAGraph()
    state["i"] = 0
    with torch.cuda.graph(g, stream=s):
        m.step(tok, ctx)
    g.replay()
    s.synchronize()
    for b in bufs.values():
        b.zero_()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record(s)
    g.replay()
    e1.record(s)
    e1.synchronize()
print(f"{name} {L} layers B={B} chained={m.chained}: {e0.elapsed_time(e1) * 1e3:.1f} us per step")
t0 = None
rows = []
for key in order:
    n = 4 if key[1] == "attn" else 16
    t = bufs[key].view(-1, n).cpu().numpy()
    t = t[t[:, 0] > 0]
    if len(t) == 0:
        continue
    t0 = t[:, 0].min() if t0 is None else min(t0, t[:, 0].min())
    rows.append((key, t))
prev_exit = None
for key, t in rows:
    r = (t - t0) / 1e3
    if key[1] == "attn":
        ex = r[:, 3][t[:, 3] > 0]
        line = (f"{str(key):14s} n={len(t):4d} entry {r[:,0].min():7.2f}-{r[:,0].max():7.2f} "
                f"wait {r[:,1].min():7.2f}-{r[:,1].max():7.2f} partial {np.median(r[:,2]):7.2f} "
                f"exit {ex.min():7.2f}-{ex.max():7.2f}")
        last = ex.max()
    else:
        own = t[:, 7] > 0  # the CTAs that write y (cluster rank 0)
        line = (f"{str(key):14s} n={len(t):4d} entry {r[:,0].min():7.2f}-{r[:,0].max():7.2f} "
                f"wait {r[:,1].min():7.2f}-{r[:,1].max():7.2f} prol {np.median(r[:,2]):7.2f} "
                f"loop {np.median(r[:,3]):7.2f}/{r[:,3].max():7.2f} clw {np.median(r[:,6]):7.2f}/{r[:,6].max():7.2f} "
                f"red {np.median(r[own,7]):7.2f}/{r[own,7].max():7.2f} "
                + (f"dsync {np.median(r[own,12]):7.2f}/{r[own,12].max():7.2f}->{np.median(r[own,13]):7.2f}/{r[own,13].max():7.2f} "
                   if (t[own, 12] > 0).any() else "")
                + f"exit {r[:,4].min():7.2f}-{r[:,4].max():7.2f}")
        last = r[:, 4].max()
    gap = "" if prev_exit is None else f"  gap {r[:,0].min() - prev_exit:5.2f}"
    print(line + gap)
    prev_exit = last
