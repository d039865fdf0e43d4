"""ncu driver: sffn_forward on the first M rows of the 7B input (per-chunk cost of forward_host), after warm-up."""
import os, sys
import numpy as np
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import torch, synth
import paper_2603_23198_b200 as sffn
cfg = synth.CONFIGS["7B"]
rows = int(sys.argv[1]) if len(sys.argv) > 1 else 4096
dev = lambda x: torch.from_numpy(x.view(np.int16)).view(torch.bfloat16).cuda()
X = dev(synth.gen_x(cfg, 0, rows)); Wg, Wu, Wd = (dev(synth.gen_w(cfg, w)) for w in "gud")
ws = torch.empty(sffn.workspace_bytes(rows, cfg.K, cfg.N, cfg.T, cfg.C, "union"), dtype=torch.uint8, device="cuda")
Y = torch.empty((rows, cfg.K), dtype=torch.bfloat16, device="cuda")
for _ in range(3):
    sffn.forward(X, Wg, Wu, Wd, cfg.T, cfg.C, out=Y, workspace=ws, algo="union")
torch.cuda.synchronize()
