"""Interleaved A/B of run-time env switches of the library (read per call, e.g. SFFN_GATE_DYN=0/1): the forward
(resident inputs, L2 flushed) and forward_host (e2e) of config $CFG (default 7B), alternating the setting every
repetition.  --var V --values a,b,c sweeps one variable; --arms "A=1,B=0;A=2,B=1" sets several per arm."""
import argparse, json, os, sys
import numpy as np
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import torch
import synth
import paper_2603_23198_b200 as sffn

ap = argparse.ArgumentParser()
ap.add_argument("--var", default="SFFN_GATE_DYN")
ap.add_argument("--values", default="0,1")
ap.add_argument("--reps", type=int, default=12)
ap.add_argument("--arms", default="", help='";"-separated arms of ","-separated VAR=value settings')
ap.add_argument("--rows", type=int, default=0, help="also time the forward on the first ROWS rows")
a = ap.parse_args()
cfg = synth.CONFIGS[os.environ.get("CFG", "7B")]
M, K, N, T, C = cfg.M, cfg.K, cfg.N, cfg.T, cfg.C
Xn = synth.gen_x(cfg, p=synth.token_targets(cfg))
dev = lambda x: torch.from_numpy(x.view(np.int16)).view(torch.bfloat16).cuda()
X = dev(Xn)
Wg, Wu, Wd = (dev(synth.gen_w(cfg, w)) for w in "gud")
ws = torch.empty(sffn.workspace_bytes(M, K, N, T, C, "union"), dtype=torch.uint8, device="cuda")
Y = torch.empty((M, K), dtype=torch.bfloat16, device="cuda")
Xh = torch.from_numpy(Xn.view(np.int16)).view(torch.bfloat16).pin_memory()
Yh = torch.empty((M, K), dtype=torch.bfloat16).pin_memory()
w1 = sffn.workspace_bytes(4096, K, N, T, C, "union")
wsh = torch.empty((w1 + 1023) // 1024 * 1024 + w1, dtype=torch.uint8, device="cuda")
flush = torch.empty(128 * 1024 * 1024, dtype=torch.float32, device="cuda")
vals = a.arms.split(";") if a.arms else a.values.split(",")


def setenv(v):
    if a.arms:
        for kv in v.split(","):
            k, x = kv.split("=")
            os.environ[k] = x
    else:
        os.environ[a.var] = v
arms = {"forward": lambda: sffn.forward(X, Wg, Wu, Wd, T, C, out=Y, workspace=ws, algo="union"),
        "e2e": lambda: sffn.forward_host(Xh, Wg, Wu, Wd, T, C, out=Yh, workspace=wsh, algo="union")}
if a.rows:
    Xr, Yr = X[:a.rows], Y[:a.rows]
    wsr = torch.empty(sffn.workspace_bytes(a.rows, K, N, T, C, "union"), dtype=torch.uint8, device="cuda")
    arms[f"forward_{a.rows}"] = lambda: sffn.forward(Xr, Wg, Wu, Wd, T, C, out=Yr, workspace=wsr, algo="union")


def once(fn):
    flush.fill_(1)
    s, e = torch.cuda.Event(True), torch.cuda.Event(True)
    s.record(); fn(); e.record(); torch.cuda.synchronize()
    return s.elapsed_time(e)


res = {(k, v): [] for k in arms for v in vals}
for v in vals:
    setenv(v)
    for f in arms.values():
        f(); f()
torch.cuda.synchronize()
for r in range(a.reps):
    for v in (vals if r % 2 == 0 else vals[::-1]):
        setenv(v)
        for k, f in arms.items():
            res[(k, v)].append(once(f))
out = {"var": a.arms or a.var, "reps": a.reps, "config": os.environ.get("CFG", "7B")}
for (k, v), t in res.items():
    out[f"{k}[{v}]_ms"] = round(float(np.median(t)), 4)
print(json.dumps(out), flush=True)
