timeout 900 python -m pytest tests -x -q -m gpu > gpurun_out/gpu_tests.log 2>&1; tail -1 gpurun_out/gpu_tests.log
for c in 3 5 4; do timeout 900 python tools/ab.py $c 3 libpfac_ref.so libpfac.so > gpurun_out/ab_c$c.log 2>&1; cat gpurun_out/ab_c$c.log; done
