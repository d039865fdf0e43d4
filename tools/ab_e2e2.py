"""PCIe floor (H2D / D2H / both, 268 MB pinned) and an interleaved A/B of host-pipeline plans (chunk rows, slots)."""
import os
import sys

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import torch  # noqa: E402

import paper_2603_23198_b200 as sffn  # noqa: E402
import synth  # noqa: E402

cfg = synth.CONFIGS["7B"]
M, K, N, T, C = cfg.M, cfg.K, cfg.N, cfg.T, cfg.C
dev = lambda x: torch.from_numpy(x.view(np.int16)).view(torch.bfloat16).cuda()
p = synth.token_targets(cfg)
Xn = synth.gen_x(cfg, p=p)
Wg, Wu, Wd = (dev(synth.gen_w(cfg, w)) for w in "gud")
Xh = torch.from_numpy(Xn.view(np.int16)).view(torch.bfloat16).pin_memory()
Yh = torch.empty((M, K), dtype=torch.bfloat16).pin_memory()
Xd = torch.empty((M, K), dtype=torch.bfloat16, device="cuda")
Yd = torch.empty((M, K), dtype=torch.bfloat16, device="cuda")
s1, s2 = torch.cuda.Stream(), torch.cuda.Stream()


def t(fn, reps=5):
    out = []
    for _ in range(reps):
        torch.cuda.synchronize()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        fn()
        e1.record()
        torch.cuda.synchronize()
        out.append(e0.elapsed_time(e1))
    return float(np.median(out))


def both():
    cur = torch.cuda.current_stream()
    s1.wait_stream(cur)
    s2.wait_stream(cur)
    with torch.cuda.stream(s1):
        Xd.copy_(Xh, non_blocking=True)
    with torch.cuda.stream(s2):
        Yh.copy_(Yd, non_blocking=True)
    cur.wait_stream(s1)
    cur.wait_stream(s2)


print(f"PCIe: H2D {t(lambda: Xd.copy_(Xh, non_blocking=True)):.3f} ms, D2H {t(lambda: Yh.copy_(Yd, non_blocking=True)):.3f} ms, "
      f"both {t(both):.3f} ms (268 MB each)")
plans = [(4096, 2), (2048, 3), (2048, 16), (4096, 9), (6144, 3)]
bufs = {}
for c, s in plans:
    n = len(sffn.forward_host_chunks(M, c))
    rows = min(c, M)
    wsz = sffn.workspace_bytes(rows, K, N, T, C)
    bufs[(c, s)] = (torch.empty((wsz + 1023) // 1024 * 1024 + wsz, dtype=torch.uint8, device="cuda"),
                    torch.empty(int(sffn.sffn.lib().sffn_forward_host_stage_bytes(K, rows)) * min(s, n) // 2,
                                dtype=torch.uint8, device="cuda"))
res = {pl: [] for pl in plans}
for rep in range(10):
    for pl in (plans if rep % 2 == 0 else plans[::-1]):
        ws, st = bufs[pl]
        res[pl].append(t(lambda: sffn.forward_host(Xh, Wg, Wu, Wd, T, C, out=Yh, workspace=ws, stage=st,
                                                   chunk_rows=pl[0], synchronize=False), reps=2))
for pl in plans:
    print(f"chunk {pl[0]:5d} slots {pl[1]:3d}: median {np.median(res[pl]):.3f} ms  mean {np.mean(res[pl]):.3f}  min {min(res[pl]):.3f}")
