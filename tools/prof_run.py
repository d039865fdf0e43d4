"""Minimal driver for ncu: one forward (pack + up_down) and one dense forward on a config, after warm-up."""
import argparse, os, sys
import numpy as np
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import torch
import synth
import paper_2603_23198_b200 as sffn

ap = argparse.ArgumentParser()
ap.add_argument("--config", default="7B")
ap.add_argument("--iters", type=int, default=2)
ap.add_argument("--dense", action="store_true")
ap.add_argument("--algo", default="auto")
ap.add_argument("--fwd", action="store_true", help="one sffn_forward call per iteration instead of pack + up_down")
a = ap.parse_args()
cfg = synth.CONFIGS[a.config]
dev = lambda x: torch.from_numpy(x.view(np.int16)).view(torch.bfloat16).cuda()
X = dev(synth.gen_x(cfg)); Wg, Wu, Wd = (dev(synth.gen_w(cfg, w)) for w in "gud")
ws = torch.empty((cfg.M, cfg.N // cfg.C), dtype=torch.int32, device="cuda")
Y = torch.empty((cfg.M, cfg.K), dtype=torch.bfloat16, device="cuda")
udws = torch.empty(max(16, sffn.up_down_workspace_bytes(cfg.M, cfg.K, cfg.N, cfg.T, cfg.C, a.algo)), dtype=torch.uint8, device="cuda")
fws = torch.empty(sffn.workspace_bytes(cfg.M, cfg.K, cfg.N, cfg.T, cfg.C, a.algo), dtype=torch.uint8, device="cuda") if a.fwd else None
for _ in range(a.iters):
    if a.fwd:
        sffn.forward(X, Wg, Wu, Wd, cfg.T, cfg.C, out=Y, workspace=fws, algo=a.algo)
        continue
    sffn.pack(X, Wg, cfg.T, cfg.C, out=ws)
    sffn.up_down(X, ws, Wu, Wd, cfg.T, cfg.C, out=Y, workspace=udws, algo=a.algo)
if a.dense:
    wdT = sffn.transpose(Wd)
    H = torch.empty((cfg.M, cfg.N), dtype=torch.bfloat16, device="cuda")
    for _ in range(a.iters):
        sffn.dense_forward(X, Wg, Wu, wdT, h=H, out=Y)
torch.cuda.synchronize()
print("done")
