cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out/ncu13
timeout 600 ncu --set full --clock-control none --import-source on -k regex:gemm_tc -s 1 -c 1 -o gpurun_out/ncu13/gate1B -f python tools/prof_run.py --config 1B --iters 2 --fwd > gpurun_out/ncu13/prof.log 2>&1; echo "ncu rc=$?"
ncu -i gpurun_out/ncu13/gate1B.ncu-rep --page raw --csv > gpurun_out/ncu13/gate1B_raw.csv 2>/dev/null
# flush vs no flush: the bench step with and without the L2 flush between steps (interleaved)
cat > /tmp/flush_ab.py <<'PY'
import os, sys, numpy as np
sys.path.insert(0, os.getcwd())
import torch, synth, paper_2603_23198_b200 as sffn
cfg = synth.CONFIGS["7B"]; M, K, N, T, C = cfg.M, cfg.K, cfg.N, cfg.T, cfg.C
dev = lambda x: torch.from_numpy(x.view(np.int16)).view(torch.bfloat16).cuda()
p = synth.token_targets(cfg); X = dev(synth.gen_x(cfg, p=p)); Wg, Wu, Wd = (dev(synth.gen_w(cfg, w)) for w in "gud")
Y = torch.empty((M, K), dtype=torch.bfloat16, device="cuda"); ws = torch.empty(sffn.workspace_bytes(M, K, N, T, C), dtype=torch.uint8, device="cuda")
flush = torch.empty(512 * 1024 * 1024 // 4, dtype=torch.float32, device="cuda")
step = lambda: sffn.forward(X, Wg, Wu, Wd, T, C, out=Y, workspace=ws)
for _ in range(3): step()
torch.cuda.synchronize(); g = torch.cuda.CUDAGraph()
with torch.cuda.graph(g): step()
for rnd in range(3):
  for fl in (True, False):
    ev = []
    for i in range(23):
        if fl: flush.fill_(1.0)
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        a.record(); g.replay(); b.record(); ev.append((a, b))
    torch.cuda.synchronize()
    ms = [a.elapsed_time(b) for a, b in ev[3:]]
    print(f"flush={fl}: mean {np.mean(ms):.3f} median {np.median(ms):.3f} min {min(ms):.3f}")
PY
timeout 300 python /tmp/flush_ab.py 2>&1 | grep -v -i warn
