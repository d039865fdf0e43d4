"""Probe of the host-buffer pipeline: PCIe H2D / D2H bandwidth alone and concurrent, per-chunk forward time,
and sffn_forward_host end to end for several chunk sizes (7B)."""
import os, sys, time
import numpy as np
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import torch, synth
import paper_2603_23198_b200 as sffn
cfg = synth.CONFIGS["7B"]
M, K, N, T, C = cfg.M, cfg.K, cfg.N, cfg.T, cfg.C
Xn = synth.gen_x(cfg)
dev = lambda x: torch.from_numpy(x.view(np.int16)).view(torch.bfloat16).cuda()
X = dev(Xn); Wg, Wu, Wd = (dev(synth.gen_w(cfg, w)) for w in "gud")
Xh = torch.from_numpy(Xn.view(np.int16)).view(torch.bfloat16).pin_memory()
Yh = torch.empty((M, K), dtype=torch.bfloat16).pin_memory()
Yd = torch.empty((M, K), dtype=torch.bfloat16, device="cuda")
Xd = torch.empty_like(Yd)

def tim(fn, n=5):
    fn(); torch.cuda.synchronize()
    ts = []
    for _ in range(n):
        s, e = torch.cuda.Event(True), torch.cuda.Event(True)
        s.record(); fn(); e.record(); torch.cuda.synchronize(); ts.append(s.elapsed_time(e))
    return float(np.median(ts))

nb = M * K * 2
s1, s2 = torch.cuda.Stream(), torch.cuda.Stream()
print(f"H2D {nb/1e6:.0f} MB: {tim(lambda: Xd.copy_(Xh, non_blocking=True)):.3f} ms")
print(f"D2H {nb/1e6:.0f} MB: {tim(lambda: Yh.copy_(Yd, non_blocking=True)):.3f} ms")
def both():
    cur = torch.cuda.current_stream()
    s1.wait_stream(cur); s2.wait_stream(cur)
    with torch.cuda.stream(s1): Xd.copy_(Xh, non_blocking=True)
    with torch.cuda.stream(s2): Yh.copy_(Yd, non_blocking=True)
    cur.wait_stream(s1); cur.wait_stream(s2)
print(f"H2D+D2H concurrent: {tim(both):.3f} ms")
for rows in (2048, 4096, 8192):
    ws = torch.empty(sffn.workspace_bytes(rows, K, N, T, C, "union"), dtype=torch.uint8, device="cuda")
    xr, yr = X[:rows], Yd[:rows]
    t = tim(lambda: sffn.forward(xr, Wg, Wu, Wd, T, C, out=yr, workspace=ws, algo="union"))
    print(f"forward M={rows}: {t:.3f} ms  (x{M//rows} = {t*M/rows:.2f} ms)")
res = {}
wsz = sffn.workspace_bytes(16384, K, N, T, C, "union")
wsd2 = torch.empty((wsz + 1023) // 1024 * 1024 + wsz, dtype=torch.uint8, device="cuda")
chunks = [int(c) for c in os.environ.get("CHUNKS", "4096,8192,16384").split(",")]
slots = [int(c) for c in os.environ.get("SLOTS", "2").split(",")]
duals = [int(c) for c in os.environ.get("DUAL", "1").split(",")]
arms = [(c, q, d) for c in chunks for q in slots for d in duals]
stg = torch.empty(int(sffn.sffn.lib().sffn_forward_host_stage_bytes(K, max(chunks))) * max(slots) // 2,
                  dtype=torch.uint8, device="cuda")
for a in arms:
    res[a] = []
for rnd in range(4):
    for c, q, d in (arms if rnd % 2 == 0 else arms[::-1]):
        st = stg[:int(sffn.sffn.lib().sffn_forward_host_stage_bytes(K, c)) * q // 2]
        w1 = sffn.workspace_bytes(c, K, N, T, C, "union")
        wsd = wsd2 if d else wsd2[:w1]  # one workspace: a single compute stream
        res[(c, q, d)].append(tim(lambda: sffn.forward_host(Xh, Wg, Wu, Wd, T, C, out=Yh, workspace=wsd,
                                                            algo="union", chunk_rows=c, stage=st), n=3))
for c, q, d in arms:
    print(f"forward_host chunk={c} slots={q} dual={d} {sffn.forward_host_chunks(M, c)}: "
          f"median {np.median(res[(c, q, d)]):.3f} ms  {[round(x, 3) for x in res[(c, q, d)]]}")
