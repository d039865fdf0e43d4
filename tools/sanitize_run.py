"""Small invocations of every entry point, for compute-sanitizer (memcheck / racecheck / synccheck)."""
import os, sys
import numpy as np
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import torch, synth
import paper_2603_23198_b200 as sffn
cfg = synth.CONFIGS["1B"].replace(M=260, K=256, N=1024, Kb=16, sparsity=0.95)
dev = lambda x: torch.from_numpy(x.view(np.int16)).view(torch.bfloat16).cuda()
X = dev(synth.gen_x(cfg)); Wg, Wu, Wd = (dev(synth.gen_w(cfg, w)) for w in "gud")
ov = torch.zeros(1, dtype=torch.int32, device="cuda")
tw = sffn.pack(X, Wg, 256, 8, overflow=ov)
sffn.unpack(tw, cfg.N, 256, 8)
for algo in ("gather", "union"):
    sffn.up_down(X, tw, Wu, Wd, 256, 8, algo=algo)
    sffn.forward(X, Wg, Wu, Wd, 256, 8, algo=algo)
    sffn.forward_nongated(X, Wg, Wd, 256, 8, algo=algo)
    sffn.forward_hybrid(X, Wg, Wu, Wd, 256, 8, backup_rows=128, algo=algo)
sffn.dense_forward(X, Wg, Wu, sffn.transpose(Wd))
sffn.gate_gemm_f32(X, Wg)
hyb = sffn.twell_to_hybrid(tw, cfg.N, 256, 8, ell_w=16, dense_cap=64)
hh = sffn.hybrid_sddmm(X, Wu, hyb, gate=True)
sffn.hybrid_spmm(hh, Wd)
f = lambda a: a.float().contiguous()
sffn.forward_f32(f(X), f(Wg), f(Wu), f(Wd), 256, 8)
xh = X.cpu().pin_memory()
sffn.forward_host(xh, Wg, Wu, Wd, 256, 8, chunk_rows=128)
if os.environ.get("SFFN_UNION_PAIR") != "1":  # NEXT-3 symmetric path on a 1-rank communicator
    comm = sffn.Comm(0, 1, torch.cuda.current_device())
    if comm.symmetric_init(cfg.M, cfg.K):
        comm.sharded_forward_sym(X, Wg, Wu, Wd, 256, 8, algo="union")
    torch.cuda.synchronize()
    comm.close()
torch.cuda.synchronize()
print("sanitize run done")

# the gate GEMM's optional dynamic tile scheduler (off by default)
os.environ["SFFN_GATE_DYN"] = "1"
sffn.forward(X, Wg, Wu, Wd, 256, 8, algo="union")
torch.cuda.synchronize()
os.environ["SFFN_GATE_DYN"] = "0"
print("dyn scheduler done", flush=True)
