"""Decode attention chains (8 layers) for the 7B / 65B shapes, over the split cap."""
import math, sys
from pathlib import Path
import torch
sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
from paper_2307_03738_b200.decode import GpuBackend  # noqa: E402
from paper_2307_03738_b200 import _lib  # noqa: E402
Lb = _lib.lib()
s = torch.cuda.Stream()
for (B, H, ctx) in [(1, 32, 513), (1, 64, 1025), (8, 64, 1025)]:
    L, hd = 8, 128
    qkv = torch.randn(B, 3 * H * hd, device="cuda")
    cos, sin = torch.ones(hd // 2, device="cuda"), torch.zeros(hd // 2, device="cuda")
    kc = torch.randn(L, B, H, ctx, hd, device="cuda").half()
    vc = torch.randn(L, B, H, ctx, hd, device="cuda").half()
    out = torch.empty(B, H * hd, device="cuda")
    for cap in [4, 8, 12, 16]:
        Lb.qigen_debug_attn_splits(cap)
        def f():
            for li in range(L):
                GpuBackend.attention(qkv, cos, sin, kc[li], vc[li], ctx - 1, 1 / math.sqrt(hd), out, torch.empty(0))
        with torch.cuda.stream(s):
            f(); s.synchronize()
            g = torch.cuda.CUDAGraph()
            with torch.cuda.graph(g, stream=s):
                f()
            g.replay(); s.synchronize()
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            e0.record(s)
            for _ in range(10):
                g.replay()
            e1.record(s); e1.synchronize()
        us = e0.elapsed_time(e1) / 10 / L * 1e3
        gb = 2 * B * H * ctx * hd * 2 / us / 1e3
        print(f"B={B} H={H} ctx={ctx} cap={cap}: {us:6.2f} us/layer  {gb:6.0f} GB/s", flush=True)
    Lb.qigen_debug_attn_splits(16)
