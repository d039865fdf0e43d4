"""A/B timing of the union up/down for the library named by SFFN_LIB (7B, L2 flushed)."""
import os, sys
import numpy as np
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import torch, synth
import paper_2603_23198_b200 as sffn
cfg = synth.CONFIGS[os.environ.get("CFG", "7B")]
if os.environ.get("M"):
    cfg = cfg.replace(M=int(os.environ["M"]))
dev = lambda x: torch.from_numpy(x.view(np.int16)).view(torch.bfloat16).cuda()
X = dev(synth.gen_x(cfg)); Wg, Wu, Wd = (dev(synth.gen_w(cfg, w)) for w in "gud")
tw = sffn.pack(X, Wg, cfg.T, cfg.C)
ws = torch.empty(sffn.up_down_workspace_bytes(cfg.M, cfg.K, cfg.N, cfg.T, cfg.C, "union"), dtype=torch.uint8, device="cuda")
Y = torch.empty((cfg.M, cfg.K), dtype=torch.bfloat16, device="cuda")
flush = torch.empty(256 * 1024 * 1024, dtype=torch.float32, device="cuda")
def t(fn, n=15):
    for _ in range(3): fn()
    ts = []
    for _ in range(n):
        flush.fill_(1); s, e = torch.cuda.Event(True), torch.cuda.Event(True); s.record(); fn(); e.record(); torch.cuda.synchronize(); ts.append(s.elapsed_time(e))
    return float(np.median(ts))
print(os.environ.get("SFFN_LIB", "default"), f"pack {t(lambda: sffn.pack(X, Wg, cfg.T, cfg.C, out=tw)):.3f} ms",
      f"up_down {t(lambda: sffn.up_down(X, tw, Wu, Wd, cfg.T, cfg.C, out=Y, workspace=ws, algo='union')):.3f} ms", flush=True)
if os.environ.get("KPROF"):
    from torch.profiler import profile, ProfilerActivity
    fws = torch.empty(sffn.workspace_bytes(cfg.M, cfg.K, cfg.N, cfg.T, cfg.C, "union"), dtype=torch.uint8, device="cuda")
    fn = (lambda: sffn.forward(X, Wg, Wu, Wd, cfg.T, cfg.C, out=Y, workspace=fws, algo='union')) if os.environ.get("KPROF") == "fwd" else \
         (lambda: sffn.up_down(X, tw, Wu, Wd, cfg.T, cfg.C, out=Y, workspace=ws, algo='union'))
    with profile(activities=[ProfilerActivity.CUDA]) as prof:
        for _ in range(5):
            flush.fill_(1); fn()
        torch.cuda.synchronize()
    agg = {}
    for e in prof.events():
        if e.device_type.name == "CUDA" and "Fill" not in e.name:
            agg.setdefault(e.name[:60], []).append(e.device_time_total if hasattr(e, "device_time_total") else e.cuda_time_total)
    for k, v in agg.items():
        print(f"   {k:60s} {np.mean(v):9.1f} us x{len(v)}")
