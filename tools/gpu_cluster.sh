# cluster/DSMEM tier: its parity tests, an A/B of the non-cluster kernels, the placement ablation with it
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_parity.py -q -x -k "cluster or placement" > gpurun_out/gputest_cluster.log 2>&1; echo "rc=$?" >> gpurun_out/gputest_cluster.log
AB_NO_TESTS=1 AB_CFGS="3:1024 5:1024" bash tools/ab_run.sh
timeout 900 python tools/placement.py 2 3 4 5 > gpurun_out/placement_cluster.jsonl 2>&1
