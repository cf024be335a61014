"""K-split choice for the decode GEMVs in a chain (per-op chains of 8 layers)."""
import sys
from pathlib import Path
import torch
sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
from paper_2307_03738_b200 import decode as D  # noqa: E402

L = 8
cfg = D.shrink(D.LLAMA_7B, n_layers=L)
m = D.LlamaTP(cfg, batch=1, max_ctx=513, seed=0)
h = torch.randn(1, cfg.d_model, device="cuda")
att = torch.randn(1, cfg.d_model, device="cuda")
qkvs = [torch.empty(1, 3 * cfg.d_model, device="cuda") for _ in range(L)]
gus = [torch.randn(1, 2 * cfg.ffn, device="cuda") for _ in range(L)]
s = torch.cuda.Stream()
for name in ["qkv", "o", "gu", "down"]:
    for ks in [0, 1, 2, 3, 4, 6, 8]:
        def f(ks=ks):
            for li, lay in enumerate(m.layers):
                pw = lay[name].pw
                if name == "qkv":
                    pw.gemv(h, out=qkvs[li], prologue="rmsnorm", norm_weight=lay["n1"], k_splits=ks)
                elif name == "o":
                    pw.gemv(att, out=h, accumulate=True, k_splits=ks)
                elif name == "gu":
                    pw.gemv(h, out=gus[li], prologue="rmsnorm", norm_weight=lay["n2"], k_splits=ks)
                else:
                    pw.gemv(gus[li], out=h, accumulate=True, prologue="swiglu", k_splits=ks)
        try:
            with torch.cuda.stream(s):
                f(); s.synchronize()
                g = torch.cuda.CUDAGraph()
                with torch.cuda.graph(g, stream=s):
                    f()
                for _ in range(3):
                    g.replay()
                e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
                e0.record(s)
                for _ in range(20):
                    g.replay()
                e1.record(s); e1.synchronize()
            print(f"{name:5s} k_splits={ks}: {e0.elapsed_time(e1) / 20 / L * 1e3:7.2f} us", flush=True)
        except Exception as e:  # noqa: BLE001
            print(f"{name:5s} k_splits={ks}: {str(e)[:60]}", flush=True)
