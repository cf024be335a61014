"""Run a few eager decode steps of a shrunk LLaMA (for ncu launch lists):
python tools/decode_breakdown.py {7b|65b} n_layers batch ctx"""
import sys
from pathlib import Path

import torch

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
from paper_2307_03738_b200 import decode as D  # noqa: E402

base = D.LLAMA_65B if (len(sys.argv) > 1 and sys.argv[1] == "65b") else D.LLAMA_7B
nl = int(sys.argv[2]) if len(sys.argv) > 2 else 2
batch = int(sys.argv[3]) if len(sys.argv) > 3 else 1
ctx = int(sys.argv[4]) if len(sys.argv) > 4 else 512
cfg = D.shrink(base, n_layers=nl)
m = D.LlamaTP(cfg, batch=batch, max_ctx=ctx + 1, seed=0)
tok = torch.zeros(batch, dtype=torch.long, device="cuda")
for _ in range(3):
    m.step(tok, ctx)
torch.cuda.synchronize()
print("ok")
