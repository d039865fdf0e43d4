"""Timings of the non-headline entry points on a BASELINE config; one JSON line.
CUDA events on the launching stream, L2 flushed between reps, median of reps."""
import argparse, json, os, sys
import numpy as np
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import torch
import synth
import paper_2603_23198_b200 as sffn

ap = argparse.ArgumentParser()
ap.add_argument("--config", default="7B")
ap.add_argument("--reps", type=int, default=10)
a = ap.parse_args()
cfg = synth.CONFIGS[a.config]
M, K, N, T, C = cfg.M, cfg.K, cfg.N, cfg.T, cfg.C
dev = lambda x: torch.from_numpy(x.view(np.int16)).view(torch.bfloat16).cuda()
p = synth.token_targets(cfg)
X = dev(synth.gen_x(cfg, p=p)); Wg, Wu, Wd = (dev(synth.gen_w(cfg, w)) for w in "gud")
flush = torch.empty(128 * 1024 * 1024, dtype=torch.float32, device="cuda")

def t(fn):
    for _ in range(3): fn()
    ts = []
    for _ in range(a.reps):
        flush.fill_(1)
        s, e = torch.cuda.Event(True), torch.cuda.Event(True)
        s.record(); fn(); e.record(); torch.cuda.synchronize(); ts.append(s.elapsed_time(e))
    return float(np.median(ts))

res = {"config": cfg.name, "M": M, "K": K, "N": N}
ws = torch.empty(sffn.workspace_bytes(M, K, N, T, C), dtype=torch.uint8, device="cuda")
Y = torch.empty((M, K), dtype=torch.bfloat16, device="cuda")
res["forward_union_ms"] = t(lambda: sffn.forward(X, Wg, Wu, Wd, T, C, out=Y, workspace=ws))
# non-gated variant: the gate statistics drive relu(x W_u) (W_g plays W_u)
res["nongated_union_ms"] = t(lambda: sffn.forward_nongated(X, Wg, Wd, T, C, out=Y, workspace=ws))
res["nongated_gather_ms"] = t(lambda: sffn.forward_nongated(X, Wg, Wd, T, C, out=Y, workspace=ws, algo="gather"))
R = M // 8
hws = torch.empty(int(sffn.sffn.lib().sffn_hybrid_workspace_bytes(M, K, N, T, C, 0, R)), dtype=torch.uint8, device="cuda")
cnt = torch.zeros(1, dtype=torch.int32, device="cuda")
res["hybrid_forward_ms"] = t(lambda: sffn.forward_hybrid(X, Wg, Wu, Wd, T, C, backup_rows=R, out=Y, workspace=hws,
                                                         backup_count=cnt))
res["hybrid_backup_rows_used"] = int(cnt.item())
tw = sffn.pack(X, Wg, T, C)
ELL_W = 384  # ~2.7x the mean row occupancy: the heavy-tailed rows beyond it fit the M/8 dense tail (P:1611 sizing)
res["hybrid_ell_w"] = ELL_W
res["twell_to_hybrid_ms"] = t(lambda: sffn.twell_to_hybrid(tw, N, T, C, ell_w=ELL_W, dense_cap=M // 8))
h = sffn.twell_to_hybrid(tw, N, T, C, ell_w=ELL_W, dense_cap=M // 8)
res["twell_to_hybrid_l0_l1"] = h["l0l1"].cpu().tolist()
res["twell_to_hybrid_dense_rows"] = int(h["dense_count"].item())
# training forward on the hybrid format (NEXT-4): SDDMM h = h_g (.) x W_u on the pattern, SpMM y = h W_d
hws2 = torch.empty(int(sffn.sffn.lib().sffn_hybrid_mm_workspace_bytes(M // 8, K, N)), dtype=torch.uint8, device="cuda")
hh = sffn.hybrid_sddmm(X, Wu, h, gate=True, workspace=hws2)
res["hybrid_sddmm_ms"] = t(lambda: sffn.hybrid_sddmm(X, Wu, h, gate=True, workspace=hws2))
res["hybrid_spmm_ms"] = t(lambda: sffn.hybrid_spmm(hh, Wd, out=Y, workspace=hws2))
res["hybrid_train_fwd_ms"] = res["twell_to_hybrid_ms"] + res["hybrid_sddmm_ms"] + res["hybrid_spmm_ms"]
res["pack_ms"] = t(lambda: sffn.pack(X, Wg, T, C, out=tw))
res["paper_design_train_fwd_ms"] = res["pack_ms"] + res["hybrid_train_fwd_ms"]
# the same outputs (Y, h_g and h in the hybrid format) through the union tensor-core path in one call
res["forward_train_union_ms"] = t(lambda: sffn.forward_train(X, Wg, Wu, Wd, T, C, ell_w=ELL_W, dense_cap=M // 8,
                                                             out=Y, workspace=ws))
# NEXT-3 on a 1-rank communicator (one GPU): the cost the reduction machinery adds to the forward when there is
# nothing to reduce — symmetric window + reduction kernel + copy-out vs the same reduction fused into the DOWN GEMM
comm = sffn.Comm(0, 1, torch.cuda.current_device())
if comm.symmetric_init(M, K):
    res["sym_1rank_ms"] = t(lambda: comm.sharded_forward_sym(X, Wg, Wu, Wd, T, C, out=Y, workspace=ws, algo="union"))
    res["fused_1rank_ms"] = t(lambda: comm.sharded_forward_fused(X, Wg, Wu, Wd, T, C, out=Y, workspace=ws))
    res["forward_union_ms_again"] = t(lambda: sffn.forward(X, Wg, Wu, Wd, T, C, out=Y, workspace=ws))
comm.close()
# fp32 mode (correctness mode; SIMT fp32 GEMM) on a row slice to bound the time
Mf = min(M, 4096)
Xf = torch.from_numpy(synth.gen_x(cfg, 0, Mf, dtype="f32", p=p)).cuda()
Wgf, Wuf, Wdf = (torch.from_numpy(synth.gen_w(cfg, w, dtype="f32")).cuda() for w in "gud")
res["fp32_forward_ms_rows"] = Mf
res["fp32_forward_ms"] = t(lambda: sffn.forward_f32(Xf, Wgf, Wuf, Wdf, T, C))
res["fp32_gate_tflops"] = 2.0 * Mf * K * N / (t(lambda: sffn.pack_f32(Xf, Wgf, T, C)) * 1e-3) / 1e12
print(json.dumps(res), flush=True)
