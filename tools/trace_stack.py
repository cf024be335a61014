"""Timeline of the persistent decode stack (csrc/decode_stack.cu): per grid
barrier, when the CTAs arrive and pass (globaltimer, us), i.e. per phase the
prologue + compute time, the arrival spread and the barrier latency.

  python tools/trace_stack.py [7b|65b] [layers] [sss depth ksl]
"""
import sys
from pathlib import Path

import numpy as np
import torch

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
from paper_2307_03738_b200 import decode as D  # noqa: E402
from paper_2307_03738_b200 import _lib  # noqa: E402

name = sys.argv[1] if len(sys.argv) > 1 else "7b"
L = int(sys.argv[2]) if len(sys.argv) > 2 else 4
Lb = _lib.lib()
if len(sys.argv) > 5:
    Lb.qigen_debug_stack_tuning(int(sys.argv[3]), int(sys.argv[4]), int(sys.argv[5]))
import os
Lb.qigen_debug_stack_mode(int(os.environ.get("STACK_MODE", "0")))  # (pf MB + 1) << 8 | mode
base, ctx = (D.LLAMA_7B, 512) if name == "7b" else (D.LLAMA_65B, 1024)
cfg = D.shrink(base, n_layers=L)
m = D.LlamaTP(cfg, batch=1, max_ctx=ctx + 1, seed=0, stack=True, keep_logits=False)
assert m.stack is not None, m.stack_reason
import ctypes
gi, dp, sm = ctypes.c_int(), ctypes.c_int(), ctypes.c_int()
Lb.qigen_decode_stack_info(m.stack, ctypes.byref(gi), ctypes.byref(dp), ctypes.byref(sm))
G = gi.value
print(f"{name} {L} layers: grid {G}, ring depth*100 + stage supersteps*10 + K slabs {dp.value}, smem {sm.value} B")
tok = torch.tensor([3], device="cuda")
nbar = 5 * L
buf = torch.zeros(nbar * G * 4, dtype=torch.int64, device="cuda")
for _ in range(3):
    m.step(tok, ctx)
torch.cuda.synchronize()
# timed without the trace
ev = [torch.cuda.Event(enable_timing=True) for _ in range(2)]
g = torch.cuda.CUDAGraph()
s = torch.cuda.Stream()
s.wait_stream(torch.cuda.current_stream())
with torch.cuda.stream(s):
    with torch.cuda.graph(g, stream=s):
        m.step(tok, ctx)
    for _ in range(5):
        g.replay()
    ev[0].record(s)
    for _ in range(50):
        g.replay()
    ev[1].record(s)
    s.synchronize()
print(f"step (graph, incl. embedding + LM head): {ev[0].elapsed_time(ev[1]) / 50 * 1e3:.1f} us")
Lb.qigen_debug_trace(buf.data_ptr())
m.step(tok, ctx)
torch.cuda.synchronize()
Lb.qigen_debug_trace(None)
assert m.stack_error() == 0
t = buf.cpu().numpy().reshape(nbar, G, 4).astype(np.float64) / 1e3
t0 = t[0, :, 2].min()
names = ["qkv", "attn", "o", "gu", "down"]
# stamps per phase and CTA: [0] outputs stored, [2] prologue done (attention: q ready),
# [3] GEMV loop done (attention: KV loop done); all relative to the previous phase's last store
tot = {}
prev = 0.0
for b in range(nbar):
    ph = names[b % 5]
    end = t[b, :, 0] - t0
    live = t[b, :, 2] > 0  # CTAs that took part (attention: idle CTAs have no stamp)
    pro = (t[b, live, 2] - t0).max() - prev
    loop = (t[b, live, 3] - t0).max() - prev
    work = end.max() - prev
    tot.setdefault(ph, []).append((work, pro, loop, end.max() - end[live].min()))
    if b < 10 or b >= nbar - 5:
        print(f"L{b // 5} {ph:5s} stored {end[live].min():8.2f}-{end.max():8.2f}  phase {work:6.2f}  "
              f"prologue {pro:5.2f}  loop done {loop:5.2f}")
    prev = end.max()
print("mean per phase (us, since the previous phase's last store): phase, prologue done, loop done, "
      "spread of the stores")
s_all = 0.0
for ph in names:
    a = np.array(tot[ph])
    s_all += a[:, 0].mean()
    print(f"  {ph:5s} {a[:, 0].mean():6.2f} {a[:, 1].mean():6.2f} {a[:, 2].mean():6.2f} {a[:, 3].mean():5.2f}")
print(f"  layer total {s_all:.2f} us")
