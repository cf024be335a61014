"""Timeline of a 7B decode layer chain (per GEMV: CTA entry, PDL wait, prologue,
loop end, exit; globaltimer, us relative to the first entry)."""
import math
import sys
from pathlib import Path
import numpy as np
import torch
sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
from paper_2307_03738_b200 import decode as D  # noqa: E402
from paper_2307_03738_b200 import _lib  # noqa: E402

L = 4
cfg = D.shrink(D.LLAMA_7B, n_layers=L)
m = D.LlamaTP(cfg, batch=1, max_ctx=513, seed=0)
pos = 512
h = torch.randn(1, cfg.d_model, device="cuda")
att = torch.empty(1, cfg.d_model, device="cuda")
be = m.backend
cos, sin = m.cos[pos], m.sin[pos]
qkvs = [torch.empty(1, 3 * cfg.d_model, device="cuda") for _ in range(L)]
gus = [torch.empty(1, 2 * cfg.ffn, device="cuda") for _ in range(L)]
Lb = _lib.lib()
import os
Lb.qigen_debug_prefetch(int(os.environ.get('PRE', '-1')))
Lb.qigen_debug_early_trigger(int(os.environ.get('EARLY', '0')))
bufs = {}


cbufs = {}
abufs = {}


def tr(key):
    b = bufs.setdefault(key, torch.zeros(4096 * 16, dtype=torch.int64, device="cuda"))
    c = cbufs.setdefault(key, torch.zeros(4096 * 16, dtype=torch.int64, device="cuda"))
    Lb.qigen_debug_trace(b.data_ptr())
    Lb.qigen_debug_trace_clk(c.data_ptr())


def full():
    for li, lay in enumerate(m.layers):
        tr((li, "qkv")); lay["qkv"](h, out=qkvs[li], prologue="rmsnorm", norm_weight=lay["n1"])
        Lb.qigen_debug_trace(None); Lb.qigen_debug_trace_clk(None)
        ab = abufs.setdefault(li, torch.zeros(4096 * 4, dtype=torch.int64, device="cuda"))
        Lb.qigen_debug_attn_trace(ab.data_ptr())
        be.attention(qkvs[li], cos, sin, m.k_cache[li], m.v_cache[li], pos, 1 / math.sqrt(128), att, m.attn_ws)
        Lb.qigen_debug_attn_trace(None)
        tr((li, "o")); lay["o"](att, out=h, accumulate=True)
        tr((li, "gu")); lay["gu"](h, out=gus[li], prologue="rmsnorm", norm_weight=lay["n2"])
        tr((li, "down")); lay["down"](gus[li], out=h, accumulate=True, prologue="swiglu")
        Lb.qigen_debug_trace(None); Lb.qigen_debug_trace_clk(None)


s = torch.cuda.Stream()
with torch.cuda.stream(s):
    full(); s.synchronize()
    g = torch.cuda.CUDAGraph()
    with torch.cuda.graph(g, stream=s):
        full()
    g.replay(); s.synchronize()
    for b in list(bufs.values()) + list(abufs.values()):
        b.zero_()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record(s); g.replay(); e1.record(s); e1.synchronize()
print(f"{L} layers: {e0.elapsed_time(e1) * 1e3:.1f} us")
t0 = min(int(b.view(-1, 16)[:, 0][b.view(-1, 16)[:, 0] > 0].min()) for b in bufs.values())
for key in sorted(bufs, key=lambda k: int(bufs[k].view(-1, 16)[:, 0][bufs[k].view(-1, 16)[:, 0] > 0].min())):
    t = bufs[key].view(-1, 16).cpu().numpy()
    t = t[t[:, 0] > 0]
    r = (t - t0) / 1e3
    print(f"{str(key):14s} n={len(t):4d} entry {r[:,0].min():7.2f}-{r[:,0].max():7.2f} wait {r[:,1].min():7.2f}-{r[:,1].max():7.2f} "
          f"prol {np.median(r[:,2]):7.2f} loop {np.median(r[:,3]):7.2f}/{r[:,3].max():7.2f} exit {r[:,4].min():7.2f}-{r[:,4].max():7.2f}")

print("entry -> before wait -> after wait (SM cycles, median):")
for key in [(3, "qkv"), (3, "o"), (3, "gu"), (3, "down")]:
    t = cbufs[key].view(-1, 16).cpu().numpy()
    t = t[t[:, 0] > 0].astype(np.int64)
    print(key, f"setup {np.median(t[:, 9] - t[:, 0]):.0f}  wait {np.median(t[:, 1] - t[:, 9]):.0f}")
print("phases in SM cycles after the PDL wait (median): xload dig1 digits sync stage0 loop exit")
for key in [(3, "qkv"), (3, "o"), (3, "gu"), (3, "down")]:
    t = cbufs[key].view(-1, 16).cpu().numpy()
    t = t[t[:, 0] > 0].astype(np.int64)
    print(key, "  ".join(f"{np.median(t[:, i] - t[:, 1]):.0f}" for i in (8, 11, 10, 2, 5, 3, 4)))

for li, ab in abufs.items():
    t = ab.view(-1, 4).cpu().numpy()
    t = t[t[:, 0] > 0]
    r = (t - t0) / 1e3
    ex = r[:, 3][t[:, 3] > 0]
    print(f"attn {li}: n={len(t)} entry {r[:,0].min():7.2f}-{r[:,0].max():7.2f} wait {r[:,1].min():7.2f}-{r[:,1].max():7.2f} "
          f"partial done {np.median(r[:,2]):7.2f}/{r[:,2].max():7.2f} combine exit {ex.min():7.2f}-{ex.max():7.2f}")
