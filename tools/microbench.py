"""Per-matrix GEMV timing (CUDA events, back-to-back launches over R rotating
copies so the working set exceeds L2).  Used for tuning; not the bench."""
import argparse
import json
import sys
from pathlib import Path

import torch

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
import paper_2307_03738_b200 as q  # noqa: E402

ap = argparse.ArgumentParser()
ap.add_argument("--shapes", default="4096x4096")
ap.add_argument("--bits", default="4")
ap.add_argument("--groups", default="128")
ap.add_argument("--splits", default="0")
ap.add_argument("--tokens", default="1")
ap.add_argument("--reps", type=int, default=50)
ap.add_argument("--graph", action="store_true")
ap.add_argument("--group", action="store_true", help="the R copies as one GemvGroup launch (tokens <= 2)")
ap.add_argument("--gmode", type=lambda v: int(v, 0), default=0, help="qigen_debug_group_mode (1: stream only)")
ap.add_argument("--x-ready", action="store_true", help="independent GEMVs (QIGEN_GEMV_X_READY)")
ap.add_argument("--wpc", type=int, default=8, help="qigen_debug_gemv_tuning: warps per CTA (8 or 16)")
args = ap.parse_args()
dev = torch.device("cuda")
q._lib.lib().qigen_debug_group_mode(args.gmode)
q._lib.lib().qigen_debug_gemv_tuning(0, args.wpc, 0, 0)
res = []
for shp in args.shapes.split(","):
    K, N = map(int, shp.split("x"))
    for b in map(int, args.bits.split(",")):
        for gs in args.groups.split(","):
            g = None if gs == "fc" else int(gs)
            cfg = q.QuantConfig(b, g)
            pw0 = q.PanelWeights.from_float(torch.randn(K, N, device=dev) * 0.02, cfg)
            nbytes = pw0.nbytes_algorithmic()
            R = max(2, int(4 * 126e6 // nbytes) + 1)
            pws = [pw0] + [q.PanelWeights(pw0.qw.clone(), pw0.qsz.clone(), K, N, cfg) for _ in range(R - 1)]
            for T in map(int, args.tokens.split(",")):
                x = torch.randn(T, K, device=dev)
                y = torch.empty(T, N, device=dev)
                for ks in map(int, args.splits.split(",")):
                    if args.group:
                        ys = torch.empty(R, T, N, device=dev)
                        grp = q.GemvGroup([(pw, x, ys[i]) for i, pw in enumerate(pws)])
                        run = grp.run
                    else:
                        def run():
                            for pw in pws:
                                pw.gemv(x, out=y, k_splits=ks, x_ready=args.x_ready)
                    try:
                        run(); torch.cuda.synchronize()
                    except Exception as e:  # noqa: BLE001 (split does not fit)
                        print(json.dumps(dict(K=K, N=N, bits=b, g=gs, tokens=T, splits=ks, err=str(e)[:50])))
                        continue
                    if args.graph:
                        gph = torch.cuda.CUDAGraph()
                        with torch.cuda.graph(gph):
                            run()
                        fn = gph.replay
                    else:
                        fn = run
                    fn(); torch.cuda.synchronize()
                    e0 = torch.cuda.Event(enable_timing=True); e1 = torch.cuda.Event(enable_timing=True)
                    e0.record()
                    for _ in range(args.reps):
                        fn()
                    e1.record(); e1.synchronize()
                    us = e0.elapsed_time(e1) * 1e3 / (args.reps * R)
                    r = dict(K=K, N=N, bits=b, g=gs, tokens=T, splits=ks, us=round(us, 2),
                             gbs=round(nbytes / us / 1e3, 1))
                    res.append(r)
                    print(json.dumps(r), flush=True)
