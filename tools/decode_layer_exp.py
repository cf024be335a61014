"""Per-layer decode cost split: CUDA graphs of L layers' worth of (a) the full
layer, (b) its 4 GEMVs only, (c) single GEMV types, (d) attention only."""
import math
import sys
from pathlib import Path
import torch
sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
from paper_2307_03738_b200 import decode as D  # noqa: E402
from paper_2307_03738_b200 import _lib  # noqa: E402

L = 8
cfg = D.shrink(D.LLAMA_7B, n_layers=L)
m = D.LlamaTP(cfg, batch=1, max_ctx=513, seed=0)
pos = 512
h = torch.randn(1, cfg.d_model, device="cuda")
att = torch.empty(1, cfg.d_model, device="cuda")
be = m.backend
cos, sin = m.cos[pos], m.sin[pos]
qkvs = [torch.empty(1, 3 * cfg.d_model, device="cuda") for _ in range(L)]
gus = [torch.empty(1, 2 * cfg.ffn, device="cuda") for _ in range(L)]


def full(pf=False):
    for li, lay in enumerate(m.layers):
        lay["qkv"](h, out=qkvs[li], prologue="rmsnorm", norm_weight=lay["n1"])
        be.attention(qkvs[li], cos, sin, m.k_cache[li], m.v_cache[li], pos, 1 / math.sqrt(128), att, m.attn_ws)
        lay["o"](att, out=h, accumulate=True)
        lay["gu"](h, out=gus[li], prologue="rmsnorm", norm_weight=lay["n2"])
        lay["down"](gus[li], out=h, accumulate=True, prologue="swiglu")


def full_folded():
    for li, lay in enumerate(m.layers):
        lay["qkv"](h, out=qkvs[li], prologue="rmsnorm_folded")
        be.attention(qkvs[li], cos, sin, m.k_cache[li], m.v_cache[li], pos, 1 / math.sqrt(128), att, m.attn_ws)
        lay["o"](att, out=h, accumulate=True)
        lay["gu"](h, out=gus[li], prologue="rmsnorm_folded")
        lay["down"](gus[li], out=h, accumulate=True, prologue="swiglu")


def gemvs():
    for li, lay in enumerate(m.layers):
        lay["qkv"](h, out=qkvs[li], prologue="rmsnorm", norm_weight=lay["n1"])
        lay["o"](att, out=h, accumulate=True)
        lay["gu"](h, out=gus[li], prologue="rmsnorm", norm_weight=lay["n2"])
        lay["down"](gus[li], out=h, accumulate=True, prologue="swiglu")


def one(name, **kw):
    def f():
        for li, lay in enumerate(m.layers):
            x = {"qkv": h, "o": att, "gu": h, "down": gus[li]}[name]
            out = {"qkv": qkvs[li], "o": h, "gu": gus[li], "down": h}[name]
            lay[name](x, out=out, **kw)
    return f


def attn():
    for li in range(L):
        be.attention(qkvs[li], cos, sin, m.k_cache[li], m.v_cache[li], pos, 1 / math.sqrt(128), att, m.attn_ws)


import os
Lb = _lib.lib()
s = torch.cuda.Stream()
def base():
    full(pf=False)
variants = [("full layer", base), ("full layer, folded RMSNorm", full_folded)]
def early():
    Lb.qigen_debug_early_trigger(1)
    full(pf=False)
    Lb.qigen_debug_early_trigger(0)
variants.append(("early trigger", early))
def normprep():
    Lb.qigen_debug_norm_prep(1)
    full(pf=False)
    Lb.qigen_debug_norm_prep(0)
variants.append(("norm prep always", normprep))
for pre in [0, 1, 2]:
    def fp(pre=pre):
        Lb.qigen_debug_prefetch(pre)
        full(pf=False)
        Lb.qigen_debug_prefetch(-1)
    variants.append((f"pre-wait stages {pre}", fp))
for ms in []:
    def f(ms=ms):
        Lb.qigen_debug_max_split(ms)
        full(pf=False)
        Lb.qigen_debug_max_split(16)
    variants.append((f"max split {ms}", f))
if os.environ.get("ALL"):
  variants += [("4 gemvs", gemvs),
                 ("qkv (rmsnorm)", one("qkv", prologue="rmsnorm", norm_weight=m.layers[0]["n1"])),
                 ("qkv (rmsnorm folded)", one("qkv", prologue="rmsnorm_folded")),
                 ("gate_up (rmsnorm folded)", one("gu", prologue="rmsnorm_folded")),
                 ("o (acc)", one("o", accumulate=True)),
                 ("gate_up (rmsnorm)", one("gu", prologue="rmsnorm", norm_weight=m.layers[0]["n2"])),
                 ("down (swiglu, acc)", one("down", prologue="swiglu", accumulate=True)),
                 ("attention", attn)]
for name, fn in variants:
    with torch.cuda.stream(s):
        fn(); s.synchronize()
        g = torch.cuda.CUDAGraph()
        with torch.cuda.graph(g, stream=s):
            fn()
        for _ in range(3):
            g.replay()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record(s)
        for _ in range(20):
            g.replay()
        e1.record(s); e1.synchronize()
    print(f"{name:22s} {e0.elapsed_time(e1) / 20 / L * 1e3:7.2f} us per layer")
