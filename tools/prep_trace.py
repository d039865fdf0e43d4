"""Per-CTA phase timeline of the union prep kernel (SFFN_PREP_TRACE=1): sort, OR pass, union build, gate lists, X copy.
Prints per-phase medians / maxima over CTAs and the kernel span (globaltimer ns)."""
import ctypes, os, sys
os.environ["SFFN_PREP_TRACE"] = "1"
import numpy as np
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import torch, synth
import paper_2603_23198_b200 as sffn
cfg = synth.CONFIGS[sys.argv[1] if len(sys.argv) > 1 else "7B"]
if len(sys.argv) > 2:
    cfg = cfg.replace(M=int(sys.argv[2]))  # e.g. one host-pipeline chunk
dev = lambda x: torch.from_numpy(x.view(np.int16)).view(torch.bfloat16).cuda()
X = dev(synth.gen_x(cfg)); Wg, Wu, Wd = (dev(synth.gen_w(cfg, w)) for w in "gud")
for _ in range(3):
    Y = sffn.forward(X, Wg, Wu, Wd, cfg.T, cfg.C, algo="union")
torch.cuda.synchronize()
lib = sffn.sffn.lib()
lib.sffn__prep_trace.argtypes = [ctypes.c_void_p, ctypes.c_int64]
lib.sffn__prep_trace.restype = ctypes.c_int64
buf = np.zeros(8 * 4096, dtype=np.uint64)
n = lib.sffn__prep_trace(buf.ctypes.data, buf.size)
tr = buf[:n].reshape(-1, 8).astype(np.int64)
tr = tr[tr[:, 0] > 0]
t0 = tr[:, 0].min()
names = ["start", "sorted", "OR pass", "built", "gate lists", "X copy end"]
print(f"{len(tr)} CTAs, span {(max(tr[:, 4].max(), tr[:, 5].max()) - t0) / 1e3:.1f} us")
for k in range(1, 6):
    prev = tr[:, k - 1] if k < 5 else tr[:, 1]
    d = (tr[:, k] - prev) / 1e3
    print(f"{names[k]:12s} phase us: median {np.median(d):7.1f}  max {d.max():7.1f}   | end rel. start: median "
          f"{np.median(tr[:, k] - t0) / 1e3:7.1f} max {(tr[:, k] - t0).max() / 1e3:7.1f}")
print(f"CTA start rel: median {np.median(tr[:, 0] - t0) / 1e3:.1f} max {(tr[:, 0] - t0).max() / 1e3:.1f} us")
