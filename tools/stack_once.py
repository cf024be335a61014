"""A few decode steps of the persistent stack at full model width (for ncu):
python tools/stack_once.py [7b|65b] [layers] [steps]"""
import sys
from pathlib import Path

import torch

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
from paper_2307_03738_b200 import decode as D  # noqa: E402

name = sys.argv[1] if len(sys.argv) > 1 else "7b"
L = int(sys.argv[2]) if len(sys.argv) > 2 else 8
steps = int(sys.argv[3]) if len(sys.argv) > 3 else 4
base, ctx = (D.LLAMA_7B, 512) if name == "7b" else (D.LLAMA_65B, 1024)
m = D.LlamaTP(D.shrink(base, n_layers=L), batch=1, max_ctx=ctx + 1, seed=0, stack=True,
              keep_logits=False)
assert m.stack is not None, m.stack_reason
tok = torch.tensor([3], device="cuda")
for _ in range(steps):
    tok = m.step(tok, ctx)
torch.cuda.synchronize()
assert m.stack_error() == 0
print("ok", tok.item())
