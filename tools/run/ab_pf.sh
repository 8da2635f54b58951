timeout 900 python tools/ab.py 4 4 libpfac_ref.so libpfac.so > gpurun_out/ab_c4.log 2>&1; cat gpurun_out/ab_c4.log
