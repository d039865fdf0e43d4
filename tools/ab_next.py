"""Interleaved (round-robin, alternating order) timing of the §8(f) entry points against the plain forward on the
7B config: removes the power-cap drift of sequential medians (tools/bench_extras.py).  One JSON line."""
import argparse, json, os, sys
import numpy as np
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import torch
import synth
import paper_2603_23198_b200 as sffn

ap = argparse.ArgumentParser()
ap.add_argument("--reps", type=int, default=12)
a = ap.parse_args()
cfg = synth.CONFIGS["7B"]
M, K, N, T, C = cfg.M, cfg.K, cfg.N, cfg.T, cfg.C
dev = lambda x: torch.from_numpy(x.view(np.int16)).view(torch.bfloat16).cuda()
X = dev(synth.gen_x(cfg, p=synth.token_targets(cfg)))
Wg, Wu, Wd = (dev(synth.gen_w(cfg, w)) for w in "gud")
ws = torch.empty(sffn.workspace_bytes(M, K, N, T, C, "union"), dtype=torch.uint8, device="cuda")
Y = torch.empty((M, K), dtype=torch.bfloat16, device="cuda")
R = M // 8
hws = torch.empty(int(sffn.sffn.lib().sffn_hybrid_workspace_bytes(M, K, N, T, C, 0, R)), dtype=torch.uint8,
                  device="cuda")
cnt = torch.zeros(1, dtype=torch.int32, device="cuda")
ELL_W = 384
flush = torch.empty(128 * 1024 * 1024, dtype=torch.float32, device="cuda")
arms = {
    "forward": lambda: sffn.forward(X, Wg, Wu, Wd, T, C, out=Y, workspace=ws),
    "forward_hybrid": lambda: sffn.forward_hybrid(X, Wg, Wu, Wd, T, C, backup_rows=R, out=Y, workspace=hws,
                                                  backup_count=cnt),
    "forward_nongated": lambda: sffn.forward_nongated(X, Wg, Wd, T, C, out=Y, workspace=ws),
    "forward_train": lambda: sffn.forward_train(X, Wg, Wu, Wd, T, C, ell_w=ELL_W, dense_cap=M // 8, out=Y,
                                                workspace=ws),
}
for f in arms.values():
    f(); f()
torch.cuda.synchronize()
ts = {k: [] for k in arms}
for r in range(a.reps):
    for k in (list(arms) if r % 2 == 0 else list(reversed(arms))):
        flush.fill_(1)
        s, e = torch.cuda.Event(True), torch.cuda.Event(True)
        s.record(); arms[k](); e.record(); torch.cuda.synchronize()
        ts[k].append(s.elapsed_time(e))
res = {"config": cfg.name, "reps": a.reps, **{k + "_ms": round(float(np.median(v)), 4) for k, v in ts.items()},
       "hybrid_backup_rows_used": int(cnt.item())}
print(json.dumps(res), flush=True)
