"""Interleaved (round-robin) timing of sffn.forward vs the 1-rank symmetric and fused all-reduce paths on a
BASELINE config: removes the power-cap drift that sequential medians pick up.  One JSON line."""
import argparse, json, os, sys
import numpy as np
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import torch
import synth
import paper_2603_23198_b200 as sffn

ap = argparse.ArgumentParser()
ap.add_argument("--config", default="7B")
ap.add_argument("--reps", type=int, default=20)
a = ap.parse_args()
cfg = synth.CONFIGS[a.config]
M, K, N, T, C = cfg.M, cfg.K, cfg.N, cfg.T, cfg.C
dev = lambda x: torch.from_numpy(x.view(np.int16)).view(torch.bfloat16).cuda()
X = dev(synth.gen_x(cfg, p=synth.token_targets(cfg)))
Wg, Wu, Wd = (dev(synth.gen_w(cfg, w)) for w in "gud")
ws = torch.empty(sffn.workspace_bytes(M, K, N, T, C, "union"), dtype=torch.uint8, device="cuda")
Y = torch.empty((M, K), dtype=torch.bfloat16, device="cuda")
flush = torch.empty(128 * 1024 * 1024, dtype=torch.float32, device="cuda")
comm = sffn.Comm(0, 1, torch.cuda.current_device())
assert comm.symmetric_init(M, K)
arms = {"forward": lambda: sffn.forward(X, Wg, Wu, Wd, T, C, out=Y, workspace=ws, algo="union"),
        "sym_1rank": lambda: comm.sharded_forward_sym(X, Wg, Wu, Wd, T, C, out=Y, workspace=ws, algo="union"),
        "fused_1rank": lambda: comm.sharded_forward_fused(X, Wg, Wu, Wd, T, C, out=Y, workspace=ws)}
for f in arms.values():
    for _ in range(3):
        f()
ts = {k: [] for k in arms}
for r in range(a.reps):
    order = list(arms) if r % 2 == 0 else list(reversed(arms))
    for k in order:
        flush.fill_(1)
        s, e = torch.cuda.Event(True), torch.cuda.Event(True)
        s.record(); arms[k](); e.record(); torch.cuda.synchronize()
        ts[k].append(s.elapsed_time(e))
res = {"config": cfg.name, "reps": a.reps, **{k + "_ms": float(np.median(v)) for k, v in ts.items()}}
comm.close()
print(json.dumps(res), flush=True)
