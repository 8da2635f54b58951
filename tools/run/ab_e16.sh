timeout 900 python -m pytest tests -x -q -m gpu > gpurun_out/gpu_tests.log 2>&1; tail -3 gpurun_out/gpu_tests.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke.log 2>&1; echo smoke rc=$?
timeout 900 python tools/ab.py 5 3 libpfac.so+PFAC_NO_ENTRY=1 libpfac.so > gpurun_out/ab_c5.log 2>&1; cat gpurun_out/ab_c5.log
