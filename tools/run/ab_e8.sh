timeout 900 python -m pytest tests -x -q -m gpu > gpurun_out/gpu_tests.log 2>&1; tail -3 gpurun_out/gpu_tests.log
timeout 900 python tools/ab.py 3 3 libpfac.so+PFAC_NO_ENTRY8=1 libpfac.so > gpurun_out/ab_c3.log 2>&1; cat gpurun_out/ab_c3.log
