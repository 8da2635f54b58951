timeout 900 python -m pytest tests -x -q -m gpu > gpurun_out/gpu_tests.log 2>&1; tail -1 gpurun_out/gpu_tests.log
timeout 900 python tools/ab.py 4 4 libpfac_ref.so libpfac.so > gpurun_out/ab_c4.log 2>&1; cat gpurun_out/ab_c4.log
