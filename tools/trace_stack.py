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
    # per-CTA durations (mean over the CTAs that took part): own previous store -> prologue
    # done -> loop done -> outputs stored
    own_prev = (t[b - 1, :, 0] - t0) if b else np.zeros(G)
    d_pro = (t[b, live, 2] - t0 - own_prev[live]).mean()
    d_loop = (t[b, live, 3] - t[b, live, 2]).mean()
    d_tail = (t[b, live, 0] - t[b, live, 3]).mean()
    if ph == "attn":
        print(f"    attention detail (per-CTA means, us): q ready -> KV batch done (warp 0) "
              f"{(t[b, live, 1] - t[b, live, 2]).mean():.2f}, -> CTA sync + new token "
              f"{(t[b, live, 3] - t[b, live, 1]).mean():.2f}")
    tot.setdefault(ph, []).append((work, pro, loop, end.max() - end[live].min(), d_pro, d_loop, d_tail))
    if b < 10 or b >= nbar - 5:
        print(f"L{b // 5} {ph:5s} stored {end[live].min():8.2f}-{end.max():8.2f}  phase {work:6.2f}  "
              f"prologue {pro:5.2f}  loop done {loop:5.2f}")
    prev = end.max()
print("mean per phase (us): since the previous phase's LAST store: phase, prologue done, loop done; "
      "spread of the stores; per-CTA means: prologue (own previous store -> records ready), "
      "loop, tail (loop done -> outputs stored)")
s_all = 0.0
for ph in names:
    a = np.array(tot[ph])
    s_all += a[:, 0].mean()
    print(f"  {ph:5s} {a[:, 0].mean():6.2f} {a[:, 1].mean():6.2f} {a[:, 2].mean():6.2f} {a[:, 3].mean():5.2f}"
          f"   | {a[:, 4].mean():5.2f} {a[:, 5].mean():5.2f} {a[:, 6].mean():5.2f}")
print(f"  layer total {s_all:.2f} us")
if os.environ.get("PER_CTA"):
    # which CTAs finish the gate|up / qkv loops late: the same ones every layer?
    for name_, b0 in (("gu", 3), ("qkv", 0), ("down", 4)):
        endl = np.stack([t[b, :, 3] - t[b, :, 3].min() for b in range(b0, nbar, 5)])  # [layers, G]
        m = endl.mean(0)
        order = np.argsort(m)
        print(f"{name_}: loop-done lateness per CTA (us, mean over layers): min {m.min():.2f} "
              f"p50 {np.median(m):.2f} p90 {np.percentile(m, 90):.2f} max {m.max():.2f}; "
              f"std over layers (mean over CTAs) {endl.std(0).mean():.2f}")
        print("  latest CTAs:", [(int(c), round(float(m[c]), 2)) for c in order[-10:]])
        print("  earliest CTAs:", [(int(c), round(float(m[c]), 2)) for c in order[:10]])
        grp = [round(float(m[k * (G // 4):(k + 1) * (G // 4)].mean()), 2) for k in range(4)]
        print("  mean by quarter of the grid:", grp)
        smid = buf.cpu().numpy().reshape(nbar, G, 4)[0, :, 1]
        by = {}
        for c in range(G):
            by.setdefault(int(smid[c]) // 2 % 8 if False else int(smid[c]) // 20, []).append(m[c])
        print("  smid of CTA 0..7:", smid[:8].tolist(), " max smid", int(smid.max()))
        print("  mean lateness by smid // 20:", {k: round(float(np.mean(v)), 2) for k, v in sorted(by.items())})
        late = order[-12:]
        print("  smids of the latest CTAs:", sorted(int(smid[c]) for c in late))
