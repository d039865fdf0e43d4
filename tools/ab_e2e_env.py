"""Interleaved A/B of run-time switches (environment variables read per call by the library) on the host-buffer
forward (sffn_forward_host) and the device forward: python tools/ab_e2e_env.py CFG CHUNK 'A=1' 'A=0,B=2' ..."""
import os, sys
import numpy as np
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import torch, synth
import paper_2603_23198_b200 as sffn
cfg = synth.CONFIGS[sys.argv[1]]
chunk = int(sys.argv[2])
variants = [dict(kv.split("=") for kv in v.split(",") if kv) for v in sys.argv[3:]]
M, K, N, T, C = cfg.M, cfg.K, cfg.N, cfg.T, cfg.C
dev = lambda x: torch.from_numpy(x.view(np.int16)).view(torch.bfloat16).cuda()
Xn = synth.gen_x(cfg)
X = dev(Xn); Wg, Wu, Wd = (dev(synth.gen_w(cfg, w)) for w in "gud")
Xh = torch.from_numpy(Xn.view(np.int16)).view(torch.bfloat16).pin_memory()
Yh = torch.empty((M, K), dtype=torch.bfloat16).pin_memory()
rows = min(chunk, M)
wsz = sffn.workspace_bytes(rows, K, N, T, C)
ws = torch.empty((wsz + 1023) // 1024 * 1024 + wsz, dtype=torch.uint8, device="cuda")
st = torch.empty(int(sffn.sffn.lib().sffn_forward_host_stage_bytes(K, rows)), dtype=torch.uint8, device="cuda")
fws = torch.empty(sffn.workspace_bytes(M, K, N, T, C), dtype=torch.uint8, device="cuda")
Y = torch.empty((M, K), dtype=torch.bfloat16, device="cuda")
res = {i: {"e2e": [], "fwd": []} for i in range(len(variants))}
def timed(fn):
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record(); fn(); e1.record(); torch.cuda.synchronize()
    return e0.elapsed_time(e1)
for rep in range(int(os.environ.get("ROUNDS", "6"))):
    order = list(range(len(variants))) if rep % 2 == 0 else list(range(len(variants)))[::-1]
    for i in order:
        for k in set().union(*variants):
            os.environ.pop(k, None)
        os.environ.update(variants[i])
        for _ in range(2):
            e = timed(lambda: sffn.forward_host(Xh, Wg, Wu, Wd, T, C, out=Yh, workspace=ws, stage=st, chunk_rows=chunk,
                                                synchronize=False))
            f = timed(lambda: sffn.forward(X, Wg, Wu, Wd, T, C, out=Y, workspace=fws))
            if rep > 0:
                res[i]["e2e"].append(e); res[i]["fwd"].append(f)
for i, v in enumerate(variants):
    print(f"{str(v):40s} e2e median {np.median(res[i]['e2e']):.3f} min {min(res[i]['e2e']):.3f}   "
          f"forward median {np.median(res[i]['fwd']):.3f}", flush=True)
