cd $GRAFT_REPO_ROOT
cat > /tmp/e2e_one.py <<'PY'
import os, sys, numpy as np
sys.path.insert(0, os.getcwd())
import torch, synth, paper_2603_23198_b200 as sffn
cfg = synth.CONFIGS["7B"]; M, K, N, T, C = cfg.M, cfg.K, cfg.N, cfg.T, cfg.C
dev = lambda x: torch.from_numpy(x.view(np.int16)).view(torch.bfloat16).cuda()
p = synth.token_targets(cfg); Xn = synth.gen_x(cfg, p=p)
Wg, Wu, Wd = (dev(synth.gen_w(cfg, w)) for w in "gud")
Xh = torch.from_numpy(Xn.view(np.int16)).view(torch.bfloat16).pin_memory(); Yh = torch.empty((M, K), dtype=torch.bfloat16).pin_memory()
rows = 4096; wsz = sffn.workspace_bytes(rows, K, N, T, C)
ws = torch.empty((wsz + 1023) // 1024 * 1024 + wsz, dtype=torch.uint8, device="cuda")
st = torch.empty(int(sffn.sffn.lib().sffn_forward_host_stage_bytes(K, rows)), dtype=torch.uint8, device="cuda")
out = []
for i in range(14):
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record(); sffn.forward_host(Xh, Wg, Wu, Wd, T, C, out=Yh, workspace=ws, stage=st, chunk_rows=rows, synchronize=False); e1.record()
    torch.cuda.synchronize()
    if i >= 4: out.append(e0.elapsed_time(e1))
print(os.environ.get("SFFN_HOST_RAMP_MIN"), sffn.forward_host_chunks(M, rows), f"median {np.median(out):.3f} min {min(out):.3f}")
PY
for i in 1 2 3; do for R in 512 2048; do SFFN_HOST_RAMP_MIN=$R timeout 300 python /tmp/e2e_one.py 2>&1 | grep -v -i warn | tail -1; done; done
