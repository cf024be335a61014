"""Kernel-time breakdown of one decode step replayed as a CUDA graph (torch.profiler /
CUPTI): python tools/decode_profile.py {7b|65b} n_layers batch ctx.  Kernels in a PDL
chain overlap, so per-kernel durations sum to more than the step."""
import sys
from collections import defaultdict
from pathlib import Path

import torch

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
from paper_2307_03738_b200 import decode as D  # noqa: E402

base = D.LLAMA_65B if (len(sys.argv) > 1 and sys.argv[1] == "65b") else D.LLAMA_7B
nl = int(sys.argv[2]) if len(sys.argv) > 2 else 4
batch = int(sys.argv[3]) if len(sys.argv) > 3 else 1
ctx = int(sys.argv[4]) if len(sys.argv) > 4 else 512
cfg = D.shrink(base, n_layers=nl)
m = D.LlamaTP(cfg, batch=batch, max_ctx=ctx + 1, seed=0)
tok = torch.zeros(batch, dtype=torch.long, device="cuda")
s = torch.cuda.Stream()
with torch.cuda.stream(s):
    for _ in range(2):
        m.step(tok, ctx)
    s.synchronize()
    g = torch.cuda.CUDAGraph()
    with torch.cuda.graph(g, stream=s):
        m.step(tok, ctx)
    for _ in range(5):
        g.replay()
    s.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record(s)
    for _ in range(20):
        g.replay()
    e1.record(s)
    e1.synchronize()
    print(f"step {e0.elapsed_time(e1) / 20 * 1e3:.1f} us for {nl} layers")
    with torch.profiler.profile(activities=[torch.profiler.ProfilerActivity.CUDA]) as prof:
        for _ in range(5):
            g.replay()
        s.synchronize()
agg, cnt = defaultdict(float), defaultdict(int)
for ev in prof.events():
    if ev.device_type == torch.autograd.DeviceType.CUDA:
        k = ev.name.split("(")[0][:70]
        agg[k] += ev.device_time / 5
        cnt[k] += 1
for k, v in sorted(agg.items(), key=lambda kv: -kv[1]):
    print(f"{v:9.1f} us/step {cnt[k] // 5:4d}x  {k}")
