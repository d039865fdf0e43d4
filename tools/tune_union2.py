"""Interleaved A/B of union raster group sizes (drift-robust: rounds over all configs, min per config)."""
import os, sys, random
import numpy as np
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import torch, synth
import paper_2603_23198_b200 as sffn
cfg = synth.CONFIGS[os.environ.get("CFG", "7B")]
dev = lambda x: torch.from_numpy(x.view(np.int16)).view(torch.bfloat16).cuda()
X = dev(synth.gen_x(cfg)); Wg, Wu, Wd = (dev(synth.gen_w(cfg, w)) for w in "gud")
ws = torch.empty(sffn.workspace_bytes(cfg.M, cfg.K, cfg.N, cfg.T, cfg.C, "union"), dtype=torch.uint8, device="cuda")
Y = torch.empty((cfg.M, cfg.K), dtype=torch.bfloat16, device="cuda")
flush = torch.empty(256 * 1024 * 1024, dtype=torch.float32, device="cuda")
def t(fn, n=5):
    fn()
    ts = []
    for _ in range(n):
        flush.fill_(1); s, e = torch.cuda.Event(True), torch.cuda.Event(True); s.record(); fn(); e.record(); torch.cuda.synchronize(); ts.append(s.elapsed_time(e))
    return float(np.median(ts))
confs = [tuple(int(x) for x in c.split(":")) for c in os.environ.get("CONFS", "8:16,2:4,2:8,4:4,4:8,16:4,8:4").split(",")]
best = {c: 1e9 for c in confs}
hist = {c: [] for c in confs}
for rnd in range(int(os.environ.get("ROUNDS", "5"))):
    order = confs[:]
    random.Random(rnd).shuffle(order)
    for up, down in order:
        os.environ["SFFN_UP_GROUP"], os.environ["SFFN_DOWN_GROUP"] = str(up), str(down)
        v = t(lambda: sffn.forward(X, Wg, Wu, Wd, cfg.T, cfg.C, out=Y, workspace=ws, algo="union"))
        best[(up, down)] = min(best[(up, down)], v)
        hist[(up, down)].append(round(v, 3))
for c in confs:
    print(f"up_group {c[0]:3d} down_group {c[1]:3d}: forward min {best[c]:.3f} ms  rounds {hist[c]}", flush=True)
