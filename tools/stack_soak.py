"""Soak test of the persistent decode stack: many consecutive greedy steps at full
7B width (few layers) against the per-op chain, every step compared (tokens,
logits), plus a long run of graph replays checking the error word.
  python tools/stack_soak.py [steps] [layers]"""
import sys
from pathlib import Path

import torch

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
from paper_2307_03738_b200 import decode as D  # noqa: E402

steps = int(sys.argv[1]) if len(sys.argv) > 1 else 300
L = int(sys.argv[2]) if len(sys.argv) > 2 else 4
cfg = D.shrink(D.LLAMA_7B, n_layers=L)
ref = D.LlamaTP(cfg, batch=1, max_ctx=steps + 2, seed=3, stack=False)
m = D.LlamaTP(cfg, batch=1, max_ctx=steps + 2, seed=3, stack=True)
assert m.stack is not None, m.stack_reason
for mm in (ref, m):
    mm.k_cache.zero_()
    mm.v_cache.zero_()
t1 = t2 = torch.tensor([11], device="cuda")
worst = 0.0
for p in range(steps):
    t1, t2 = ref.step(t1, p), m.step(t2, p)
    l1, l2 = ref.last_logits.double(), m.last_logits.double()
    err = ((l2 - l1).abs().max() / (1 + l1.abs().max())).item()
    worst = max(worst, err)
    assert torch.equal(t1, t2), (p, err)
    assert err < 5e-4, (p, err)
assert m.stack_error() == 0
print(f"{steps} consecutive steps, {L} layers at 7B width: same tokens, worst logit error {worst:.2e}")
# many replays of one captured step
g = torch.cuda.CUDAGraph()
s = torch.cuda.Stream()
s.wait_stream(torch.cuda.current_stream())
tok = torch.tensor([5], device="cuda")
with torch.cuda.stream(s):
    m.step(tok, steps)
    l0 = m.last_logits.clone()
    with torch.cuda.graph(g, stream=s):
        m.step(tok, steps)
    for i in range(20000):
        g.replay()
    s.synchronize()
assert torch.equal(m.last_logits, l0) and m.stack_error() == 0
print("20000 graph replays: identical logits, no wait timed out")
