"""Sweep raster group sizes of the union up/down on the 7B config (CUDA events, L2 flushed)."""
import os, sys, itertools
import numpy as np
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import torch, synth
import paper_2603_23198_b200 as sffn
cfg = synth.CONFIGS[sys.argv[1] if len(sys.argv) > 1 else "7B"]
dev = lambda x: torch.from_numpy(x.view(np.int16)).view(torch.bfloat16).cuda()
X = dev(synth.gen_x(cfg)); Wg, Wu, Wd = (dev(synth.gen_w(cfg, w)) for w in "gud")
tw = sffn.pack(X, Wg, cfg.T, cfg.C)
ws = torch.empty(sffn.up_down_workspace_bytes(cfg.M, cfg.K, cfg.N, cfg.T, cfg.C, "union"), dtype=torch.uint8, device="cuda")
Y = torch.empty((cfg.M, cfg.K), dtype=torch.bfloat16, device="cuda")
flush = torch.empty(256 * 1024 * 1024, dtype=torch.float32, device="cuda")
def t(fn, n=10):
    for _ in range(3): fn()
    ts = []
    for _ in range(n):
        flush.fill_(1); s, e = torch.cuda.Event(True), torch.cuda.Event(True); s.record(); fn(); e.record(); torch.cuda.synchronize(); ts.append(s.elapsed_time(e))
    return float(np.median(ts))
for up, down in itertools.product([int(v) for v in os.environ.get("UPS", "2,4,8,16").split(",")], [int(v) for v in os.environ.get("DOWNS", "4,8,16,32,64").split(",")]):
    os.environ["SFFN_UP_GROUP"], os.environ["SFFN_DOWN_GROUP"] = str(up), str(down)
    print(f"up_group {up:4d} down_group {down:3d}: up_down {t(lambda: sffn.up_down(X, tw, Wu, Wd, cfg.T, cfg.C, out=Y, workspace=ws, algo='union')):.3f} ms", flush=True)
