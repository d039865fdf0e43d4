cd $GRAFT_REPO_ROOT
timeout 900 python -m pytest tests/test_gpu_parity.py -m gpu -q -p no:cacheprovider -x -k "union or launch or forward_host or train or full_size or all_rows or fused or sharded" > gpurun_out/pyt4.log 2>&1; echo "pytest rc=$?"; tail -3 gpurun_out/pyt4.log
timeout 300 python tools/timeline.py --config 7B > gpurun_out/timeline4.log 2>&1; grep -v -i warn gpurun_out/timeline4.log | tail -12
timeout 600 python tools/ab_e2e.py 7B > gpurun_out/ab_e2e.log 2>&1; echo "ab rc=$?"; cat gpurun_out/ab_e2e.log | grep -v -i warn
