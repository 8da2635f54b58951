timeout 600 python tools/ab.py 2 8 libpfac_ref.so libpfac.so > gpurun_out/ab_c2.log 2>&1; cat gpurun_out/ab_c2.log
