"""Interleaved A/B of several libsffn builds in ONE process: the device forward (sffn_forward, resident inputs) and
the host-buffer forward (sffn_forward_host, pinned X/Y, 4096-row chunks) — CUDA events, medians over rounds 1..R-1."""
import ctypes, os, sys
import numpy as np
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import torch, synth
libs = sys.argv[1:]
cfg = synth.CONFIGS[os.environ.get("CFG", "7B")]
M, K, N, T, C = cfg.M, cfg.K, cfg.N, cfg.T, cfg.C
dev = lambda x: torch.from_numpy(x.view(np.int16)).view(torch.bfloat16).cuda()
Xn = synth.gen_x(cfg)
X = dev(Xn); Wg, Wu, Wd = (dev(synth.gen_w(cfg, w)) for w in "gud")
Xh = torch.from_numpy(Xn.view(np.int16)).view(torch.bfloat16).pin_memory()
Yh = torch.empty((M, K), dtype=torch.bfloat16).pin_memory()
Y = torch.empty((M, K), dtype=torch.bfloat16, device="cuda")
flush = torch.empty(128 * 1024 * 1024, dtype=torch.float32, device="cuda")
vp, i64 = ctypes.c_void_p, ctypes.c_int64
L = []
R = 4096
for p in libs:
    l = ctypes.CDLL(os.path.abspath(p), mode=ctypes.RTLD_LOCAL)
    l.sffn_forward.argtypes = [vp, vp, vp, vp, i64, i64, i64, ctypes.c_int, ctypes.c_int, vp, vp, ctypes.c_size_t, vp,
                               ctypes.c_int, vp]
    l.sffn_forward_workspace_bytes.argtypes = [i64, i64, i64, ctypes.c_int, ctypes.c_int, ctypes.c_int]
    l.sffn_forward_workspace_bytes.restype = ctypes.c_size_t
    l.sffn_forward_host_stage_bytes.argtypes = [i64, i64]
    l.sffn_forward_host_stage_bytes.restype = ctypes.c_size_t
    l.sffn_forward_host.argtypes = [vp, vp, vp, vp, i64, i64, i64, ctypes.c_int, ctypes.c_int, vp, vp, ctypes.c_size_t,
                                    vp, ctypes.c_size_t, vp, ctypes.c_int, i64, vp]
    ws = torch.empty(l.sffn_forward_workspace_bytes(M, K, N, T, C, 2), dtype=torch.uint8, device="cuda")
    wsz = l.sffn_forward_workspace_bytes(R, K, N, T, C, 2)
    hws = torch.empty((wsz + 1023) // 1024 * 1024 + wsz, dtype=torch.uint8, device="cuda")
    st = torch.empty(l.sffn_forward_host_stage_bytes(K, R), dtype=torch.uint8, device="cuda")
    L.append((l, ws, hws, st))
P = lambda t: vp(t.data_ptr())
def t(fn, n=3):
    fn(); torch.cuda.synchronize()
    r = []
    for _ in range(n):
        flush.fill_(1); s, e = torch.cuda.Event(True), torch.cuda.Event(True); s.record(); fn(); e.record(); torch.cuda.synchronize(); r.append(s.elapsed_time(e))
    return float(np.median(r))
res = {i: {"fwd": [], "e2e": []} for i in range(len(L))}
for rnd in range(int(os.environ.get("ROUNDS", "6"))):
    idx = list(range(len(L)))
    if rnd % 2:
        idx.reverse()
    for i in idx:
        l, ws, hws, st = L[i]
        res[i]["fwd"].append(t(lambda: l.sffn_forward(P(X), P(Wg), P(Wu), P(Wd), M, K, N, T, C, P(Y), P(ws), ws.numel(), None, 2, None)))
        res[i]["e2e"].append(t(lambda: l.sffn_forward_host(P(Xh), P(Wg), P(Wu), P(Wd), M, K, N, T, C, P(Yh), P(hws), hws.numel(),
                                                             P(st), st.numel(), None, 2, R, None)))
for i, p in enumerate(libs):
    print(f"{p:40s} forward {np.median(res[i]['fwd'][1:]):.3f} ms  e2e {np.median(res[i]['e2e'][1:]):.3f} ms   "
          f"(e2e rounds {[round(x, 3) for x in res[i]['e2e']]})", flush=True)
