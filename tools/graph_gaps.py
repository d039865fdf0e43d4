"""Gap analysis of the bench step: replay the forward's CUDA graph under the torch profiler and compare the sum
of kernel durations with the span from the first kernel start to the last kernel end."""
import os, sys
import numpy as np
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import torch, synth
import paper_2603_23198_b200 as sffn
from torch.profiler import profile, ProfilerActivity
cfg = synth.CONFIGS[os.environ.get("CFG", "7B")]
dev = lambda x: torch.from_numpy(x.view(np.int16)).view(torch.bfloat16).cuda()
X = dev(synth.gen_x(cfg)); Wg, Wu, Wd = (dev(synth.gen_w(cfg, w)) for w in "gud")
ws = torch.empty(sffn.workspace_bytes(cfg.M, cfg.K, cfg.N, cfg.T, cfg.C, "union"), dtype=torch.uint8, device="cuda")
Y = torch.empty((cfg.M, cfg.K), dtype=torch.bfloat16, device="cuda")
step = lambda: sffn.forward(X, Wg, Wu, Wd, cfg.T, cfg.C, out=Y, workspace=ws, algo="union")
for _ in range(3): step()
torch.cuda.synchronize()
g = torch.cuda.CUDAGraph()
with torch.cuda.graph(g):
    step()
for _ in range(3): g.replay()
torch.cuda.synchronize()
with profile(activities=[ProfilerActivity.CUDA]) as prof:
    for _ in range(5):
        g.replay()
    torch.cuda.synchronize()
ev = sorted([e for e in prof.events() if e.device_type.name == "CUDA"], key=lambda e: e.time_range.start)
# split into replays by the gate GEMM (first kernel of each step)
steps, cur = [], []
for e in ev:
    if "gemm_tc_kernel" in e.name and cur:
        steps.append(cur); cur = []
    cur.append(e)
steps.append(cur)
for s in steps[1:]:
    span = s[-1].time_range.end - s[0].time_range.start
    busy = sum(e.time_range.end - e.time_range.start for e in s)
    print(f"step span {span:8.1f} us  kernels {busy:8.1f} us  gaps {span - busy:6.1f} us  ({len(s)} ops)")
