import torch,sys
sys.path.insert(0,'.')
from paper_2307_03738_b200 import decode as D
cfg=D.shrink(D.LLAMA_65B, n_layers=1)
m=D.LlamaTP(cfg,batch=1,max_ctx=1025,seed=0)
torch.cuda.synchronize(); print("init ok", flush=True)
tok=torch.zeros(1,dtype=torch.long,device="cuda")
import math
lay=m.layers[0]; h=m.embed[tok].float()
qkv=lay["qkv"](h, prologue="rmsnorm", norm_weight=lay["n1"]); torch.cuda.synchronize(); print("qkv ok", flush=True)
att=torch.empty(1, m.nh*128, device="cuda")
m.backend.attention(qkv, m.cos[1024], m.sin[1024], m.k_cache[0], m.v_cache[0], 1024, 1/math.sqrt(128), att, m.attn_ws); torch.cuda.synchronize(); print("attn ok", flush=True)
lay["o"](att, out=h, accumulate=True); torch.cuda.synchronize(); print("o ok", flush=True)
gu=lay["gu"](h, prologue="rmsnorm", norm_weight=lay["n2"]); torch.cuda.synchronize(); print("gu ok", flush=True)
lay["down"](gu, out=h, accumulate=True, prologue="swiglu"); torch.cuda.synchronize(); print("down ok", flush=True)
