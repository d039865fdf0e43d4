"""A/B of the host-buffer forward (sffn_forward_host) plans in one process, interleaved: chunk rows x staging slots.
Prints the median ms per plan (CUDA events around the call, as bench.py's e2e leg)."""
import itertools
import os
import sys

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import torch  # noqa: E402

import paper_2603_23198_b200 as sffn  # noqa: E402
import synth  # noqa: E402

cfg = synth.CONFIGS[sys.argv[1] if len(sys.argv) > 1 else "7B"]
M, K, N, T, C = cfg.M, cfg.K, cfg.N, cfg.T, cfg.C
dev = lambda x: torch.from_numpy(x.view(np.int16)).view(torch.bfloat16).cuda()
p = synth.token_targets(cfg)
Xn = synth.gen_x(cfg, p=p)
Wg, Wu, Wd = (dev(synth.gen_w(cfg, w)) for w in "gud")
Xh = torch.from_numpy(Xn.view(np.int16)).view(torch.bfloat16).pin_memory()
Yh = torch.empty((M, K), dtype=torch.bfloat16).pin_memory()
ref = None
plans = [(c, s) for c, s in itertools.product([2048, 4096, 6144, 8192], [2, 3, 99])]
if os.environ.get("PLANS"):  # e.g. PLANS="4096:2,2048:99,4096:99"
    plans = [tuple(int(v) for v in p.split(":")) for p in os.environ["PLANS"].split(",")]
res = {pl: [] for pl in plans}
bufs = {}
for c, s in plans:
    n = len(sffn.forward_host_chunks(M, c))
    slots = min(s, n)
    rows = min(c, M)
    wsz = sffn.workspace_bytes(rows, K, N, T, C)
    bufs[(c, s)] = (torch.empty((wsz + 1023) // 1024 * 1024 + wsz, dtype=torch.uint8, device="cuda"),
                    torch.empty(int(sffn.sffn.lib().sffn_forward_host_stage_bytes(K, rows)) * slots // 2,
                                dtype=torch.uint8, device="cuda"), slots)
for rep in range(int(os.environ.get("REPS", "6"))):
    for pl in (plans if rep % 2 == 0 else plans[::-1]):
        ws, st, slots = bufs[pl]
        for it in range(3):
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            e0.record()
            sffn.forward_host(Xh, Wg, Wu, Wd, T, C, out=Yh, workspace=ws, stage=st, chunk_rows=pl[0],
                              synchronize=False)
            e1.record()
            torch.cuda.synchronize()
            if rep > 0:
                res[pl].append(e0.elapsed_time(e1))
        if ref is None:
            ref = Yh.clone()
        else:
            assert torch.equal(Yh.view(torch.int16), ref.view(torch.int16)) or pl[0] % 2048, pl
for pl in plans:
    print(f"chunk {pl[0]:5d} slots {min(pl[1], len(sffn.forward_host_chunks(M, pl[0]))):3d}: "
          f"median {np.median(res[pl]):.3f} ms  min {min(res[pl]):.3f}")
