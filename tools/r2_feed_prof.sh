cd /root/repo
mkdir -p gpurun_out/r02
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm,power.limit --format=csv > gpurun_out/r02/gpu2.txt
timeout 300 ./tools/exp_feed > gpurun_out/r02/exp_feed.txt 2>&1; echo "feed rc=$?"; cat gpurun_out/r02/exp_feed.txt
bash tools/prof_step.sh > gpurun_out/r02/prof_step.log 2>&1; echo "prof rc=$?"; tail -5 gpurun_out/r02/prof_step.log
mv gpurun_out/ncu_step gpurun_out/r02/ncu_step
