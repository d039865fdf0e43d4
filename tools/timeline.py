"""Kernel timeline of the bench step (torch.profiler / CUPTI traces every kernel of the process, the library's too):
per-kernel durations, the idle gaps between consecutive kernels, and the step span — in the real step context
(graph replay after an L2 flush, as bench.py times it).  Usage: python tools/timeline.py [--config 7B] [--eager]"""
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
ap.add_argument("--eager", action="store_true")
ap.add_argument("--steps", type=int, default=3)
ap.add_argument("--algo", default="auto")
ap.add_argument("--out", default=None)
a = ap.parse_args()
cfg = synth.CONFIGS[a.config]
dev = lambda x: torch.from_numpy(x.view(np.int16)).view(torch.bfloat16).cuda()
p = synth.token_targets(cfg)
X = dev(synth.gen_x(cfg, p=p))
Wg, Wu, Wd = (dev(synth.gen_w(cfg, w)) for w in "gud")
Y = torch.empty((cfg.M, cfg.K), dtype=torch.bfloat16, device="cuda")
ws = torch.empty(sffn.workspace_bytes(cfg.M, cfg.K, cfg.N, cfg.T, cfg.C, a.algo), dtype=torch.uint8, device="cuda")
flush = torch.empty(512 * 1024 * 1024 // 4, dtype=torch.float32, device="cuda")


def step():
    sffn.forward(X, Wg, Wu, Wd, cfg.T, cfg.C, out=Y, workspace=ws, algo=a.algo)


for _ in range(3):
    step()
torch.cuda.synchronize()
fn = step
if not a.eager:
    g = torch.cuda.CUDAGraph()
    with torch.cuda.graph(g):
        step()
    fn = g.replay
for _ in range(3):
    flush.fill_(1.0)
    fn()
torch.cuda.synchronize()
# the same steps timed with CUDA events exactly as bench.py does (flush outside the events), for comparison with
# the CUPTI span below
ev_ms = []
for _ in range(20):
    flush.fill_(1.0)
    s0, s1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    s0.record()
    fn()
    s1.record()
    ev_ms.append((s0, s1))
torch.cuda.synchronize()
ev_ms = [a.elapsed_time(b) for a, b in ev_ms]
print(f"events: median {np.median(ev_ms) * 1e3:.1f} us, min {min(ev_ms) * 1e3:.1f}, max {max(ev_ms) * 1e3:.1f}")
from torch.profiler import ProfilerActivity, profile  # noqa: E402

with profile(activities=[ProfilerActivity.CUDA]) as prof:
    for _ in range(a.steps):
        flush.fill_(1.0)
        fn()
    torch.cuda.synchronize()
ev = [e for e in prof.events() if e.device_type.name == "CUDA" and e.time_range.end > e.time_range.start]
ev.sort(key=lambda e: e.time_range.start)
steps, cur = [], []
for e in ev:
    if "FillFunctor" in e.name:
        if cur:
            steps.append(cur)
        cur = []
        continue
    cur.append(e)
if cur:
    steps.append(cur)
res = []
for s in steps:
    t0 = s[0].time_range.start
    rows = []
    prev_end = t0
    for e in s:
        rows.append({"kernel": e.name.split("(")[0][-60:], "start_us": e.time_range.start - t0,
                     "dur_us": e.time_range.end - e.time_range.start, "gap_us": e.time_range.start - prev_end})
        prev_end = e.time_range.end
    res.append({"span_us": s[-1].time_range.end - t0, "busy_us": sum(r["dur_us"] for r in rows),
                "gaps_us": sum(r["gap_us"] for r in rows), "kernels": rows})
for r in res:
    print(f"step span {r['span_us']:.1f} us, kernels {r['busy_us']:.1f} us, gaps {r['gaps_us']:.1f} us")
for k in res[-1]["kernels"]:
    print(f"  {k['kernel']:60s} {k['dur_us']:9.1f} us  gap {k['gap_us']:6.1f}")
if a.out:
    json.dump(res, open(a.out, "w"), indent=1)
