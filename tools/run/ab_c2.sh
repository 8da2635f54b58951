PFAC_LIB=paper_1702_03657_b200/libpfac_ref.so timeout 120 python tools/host_launch.py 2
timeout 120 python tools/host_launch.py 2
timeout 900 python tools/ab.py 2 10 libpfac_ref.so libpfac.so > gpurun_out/ab_c2.log 2>&1; cat gpurun_out/ab_c2.log
