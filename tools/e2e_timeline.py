"""Timeline of the end-to-end host-buffer forward (sffn_forward_host: H2D / compute / D2H on three streams, row
chunks): CUPTI traces (torch.profiler) of every kernel and memcpy — how long the copy engines and the SMs are busy,
and where each is idle.  Usage: python tools/e2e_timeline.py [--config 7B] [--chunk 4096]"""
import argparse
import json
import os
import sys

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import torch  # noqa: E402

import paper_2603_23198_b200 as sffn  # noqa: E402
import synth  # noqa: E402

ap = argparse.ArgumentParser()
ap.add_argument("--config", default="7B")
ap.add_argument("--chunk", type=int, default=4096)
ap.add_argument("--out", default=None)
a = ap.parse_args()
cfg = synth.CONFIGS[a.config]
M, K, N, T, C = cfg.M, cfg.K, cfg.N, cfg.T, cfg.C
dev = lambda x: torch.from_numpy(x.view(np.int16)).view(torch.bfloat16).cuda()
p = synth.token_targets(cfg)
Xn = synth.gen_x(cfg, p=p)
Wg, Wu, Wd = (dev(synth.gen_w(cfg, w)) for w in "gud")
Xh = torch.from_numpy(Xn.view(np.int16)).view(torch.bfloat16).pin_memory()
Yh = torch.empty((M, K), dtype=torch.bfloat16).pin_memory()
rows = min(a.chunk, M)
wsz = sffn.workspace_bytes(rows, K, N, T, C)
ws = torch.empty((wsz + 1023) // 1024 * 1024 + wsz, dtype=torch.uint8, device="cuda")
stage = torch.empty(int(sffn.sffn.lib().sffn_forward_host_stage_bytes(K, ((rows + 127) // 128) * 128)),
                    dtype=torch.uint8, device="cuda")
print("chunks", sffn.forward_host_chunks(M, a.chunk))


def step():
    sffn.forward_host(Xh, Wg, Wu, Wd, T, C, out=Yh, workspace=ws, stage=stage, chunk_rows=a.chunk, synchronize=False)


for _ in range(3):
    step()
torch.cuda.synchronize()
evs = []
for _ in range(5):
    s0, s1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    s0.record()
    step()
    s1.record()
    evs.append((s0, s1))
torch.cuda.synchronize()
print("events ms:", [round(x.elapsed_time(y), 3) for x, y in evs])
from torch.profiler import ProfilerActivity, profile  # noqa: E402

with profile(activities=[ProfilerActivity.CUDA]) as prof:
    step()
    torch.cuda.synchronize()
ev = [e for e in prof.events() if e.device_type.name == "CUDA" and e.time_range.end > e.time_range.start]
ev.sort(key=lambda e: e.time_range.start)
t0 = ev[0].time_range.start
kinds = {"h2d": [], "d2h": [], "kernel": []}
rows_out = []
for e in ev:
    n = e.name
    k = "h2d" if ("HtoD" in n or "Host to Device" in n) else "d2h" if ("DtoH" in n or "Device to Host" in n) else "kernel"
    if "Memcpy" in n and k == "kernel":
        k = "dtod"
        kinds.setdefault("dtod", [])
    kinds[k].append((e.time_range.start - t0, e.time_range.end - t0))
    rows_out.append({"name": n.split("(")[0][-50:], "kind": k, "start": e.time_range.start - t0,
                     "dur": e.time_range.end - e.time_range.start})


def busy(iv):
    iv = sorted(iv)
    tot, cs, ce = 0.0, None, None
    for s, e in iv:
        if cs is None or s > ce:
            if cs is not None:
                tot += ce - cs
            cs, ce = s, e
        else:
            ce = max(ce, e)
    if cs is not None:
        tot += ce - cs
    return tot


span = max(e for v in kinds.values() for _, e in v)
print(f"span {span:.0f} us; busy: " + ", ".join(f"{k} {busy(v):.0f} us" for k, v in kinds.items()))
for r in rows_out:
    print(f"  {r['start']:9.1f} {r['dur']:8.1f}  {r['kind']:6s} {r['name']}")
if a.out:
    json.dump(rows_out, open(a.out, "w"))
