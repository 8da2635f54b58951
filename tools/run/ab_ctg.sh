set -x
timeout 900 python -m pytest tests -x -q -m gpu > gpurun_out/gpu_tests.log 2>&1; tail -3 gpurun_out/gpu_tests.log
timeout 600 python tools/ab.py 2 8 libpfac_ref.so libpfac.so > gpurun_out/ab_c2.log 2>&1; cat gpurun_out/ab_c2.log
timeout 600 python tools/ab.py 3 3 libpfac_ref.so libpfac.so libpfac.so+PFAC_CTG64=32 > gpurun_out/ab_c3.log 2>&1; cat gpurun_out/ab_c3.log
timeout 600 python tools/ab.py 5 3 libpfac_ref.so libpfac.so+PFAC_CTG64=60 > gpurun_out/ab_c5.log 2>&1; cat gpurun_out/ab_c5.log
