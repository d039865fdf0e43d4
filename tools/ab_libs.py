"""Interleaved A/B of several libsffn builds in ONE process (drift-robust): each round times sffn_pack and
sffn_forward of every library in turn on the same inputs; prints per-library medians over rounds 1..R-1."""
import ctypes, os, sys
import numpy as np
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import torch, synth
import paper_2603_23198_b200 as sffn
libs = sys.argv[1:]
cfg = synth.CONFIGS[os.environ.get("CFG", "7B")]
dev = lambda x: torch.from_numpy(x.view(np.int16)).view(torch.bfloat16).cuda()
X = dev(synth.gen_x(cfg)); Wg, Wu, Wd = (dev(synth.gen_w(cfg, w)) for w in "gud")
M, K, N, T, C = cfg.M, cfg.K, cfg.N, cfg.T, cfg.C
ws = torch.empty(sffn.workspace_bytes(M, K, N, T, C, "union"), dtype=torch.uint8, device="cuda")
tw = torch.empty((M, N // C), dtype=torch.int32, device="cuda")
Y = torch.empty((M, K), dtype=torch.bfloat16, device="cuda")
flush = torch.empty(256 * 1024 * 1024, dtype=torch.float32, device="cuda")
vp = ctypes.c_void_p
L = []
for p in libs:
    l = ctypes.CDLL(os.path.abspath(p), mode=ctypes.RTLD_LOCAL)
    l.sffn_pack.argtypes = [vp, vp, ctypes.c_int64, ctypes.c_int64, ctypes.c_int64, ctypes.c_int, ctypes.c_int, vp, vp, vp]
    l.sffn_forward.argtypes = [vp, vp, vp, vp, ctypes.c_int64, ctypes.c_int64, ctypes.c_int64, ctypes.c_int, ctypes.c_int,
                               vp, vp, ctypes.c_size_t, vp, ctypes.c_int, vp]
    L.append(l)
P = lambda t: vp(t.data_ptr())
def t(fn, n=3):
    fn(); torch.cuda.synchronize()
    r = []
    for _ in range(n):
        flush.fill_(1); s, e = torch.cuda.Event(True), torch.cuda.Event(True); s.record(); fn(); e.record(); torch.cuda.synchronize(); r.append(s.elapsed_time(e))
    return float(np.median(r))
res = {i: {"pack": [], "fwd": []} for i in range(len(L))}
for rnd in range(int(os.environ.get("ROUNDS", "6"))):
    idx = list(range(len(L)))
    if rnd % 2:
        idx.reverse()  # ABBA order: no library always runs on the hotter GPU
    for i in idx:
        l = L[i]
        res[i]["pack"].append(t(lambda: l.sffn_pack(P(X), P(Wg), M, K, N, T, C, P(tw), None, None)))
        res[i]["fwd"].append(t(lambda: l.sffn_forward(P(X), P(Wg), P(Wu), P(Wd), M, K, N, T, C, P(Y), P(ws), ws.numel(), None, 2, None)))
for i, p in enumerate(libs):
    print(f"{p:45s} pack {np.median(res[i]['pack'][1:]):.3f} ms  forward {np.median(res[i]['fwd'][1:]):.3f} ms   "
          f"(rounds pack {[round(x, 3) for x in res[i]['pack']]})", flush=True)
