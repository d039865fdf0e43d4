"""Gate GEMM role timing from a probe build (-DSFFN_GEMM_EPI_TRACE, SFFN_LIB=build/libsffn_epitrace.so): mean cycles
of a TwELL epilogue per warp and tile (accumulator full -> released), of a tile's MMA issue (accumulator free -> last
commit) and of the MMA thread's wait for a free accumulator.  argv: config (default 7B)."""
import ctypes, os, sys
import numpy as np
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import torch, synth
import paper_2603_23198_b200 as sffn
cfg = synth.CONFIGS[sys.argv[1] if len(sys.argv) > 1 else "7B"]
dev = lambda x: torch.from_numpy(x.view(np.int16)).view(torch.bfloat16).cuda()
X = dev(synth.gen_x(cfg)); Wg = dev(synth.gen_w(cfg, "g"))
tw = torch.empty((cfg.M, cfg.N // cfg.C), dtype=torch.int32, device="cuda")
lib = sffn.sffn.lib()
lib.sffn__gemm_trace.argtypes = [ctypes.c_void_p]
buf = np.zeros(8, dtype=np.uint64)
for _ in range(2):
    sffn.pack(X, Wg, cfg.T, cfg.C, out=tw)
torch.cuda.synchronize()
lib.sffn__gemm_trace(buf.ctypes.data)  # reset
s, e = torch.cuda.Event(True), torch.cuda.Event(True)
s.record(); sffn.pack(X, Wg, cfg.T, cfg.C, out=tw); e.record(); torch.cuda.synchronize()
lib.sffn__gemm_trace(buf.ctypes.data)
ep, ne, mm, nt, wt = (int(x) for x in buf[:5])
print(f"{sys.argv[1] if len(sys.argv) > 1 else '7B'}: pack {s.elapsed_time(e):.3f} ms; epilogue {ep / max(ne, 1):.0f} cyc per warp-tile "
      f"({ne} warp-tiles); MMA issue {mm / max(nt, 1):.0f} cyc per tile ({nt} tiles); MMA wait for accumulator "
      f"{wt / max(nt, 1):.0f} cyc per tile")
