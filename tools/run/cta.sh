timeout 300 python tools/cta_hist.py 5 > gpurun_out/cta_c5.log 2>&1
make -s paper_1702_03657_b200/libpfac_timing.so
PFAC_LIB=paper_1702_03657_b200/libpfac_timing.so timeout 300 python tools/timing.py 5 > gpurun_out/timing_c5.log 2>&1
PFAC_LIB=paper_1702_03657_b200/libpfac_timing.so timeout 300 python tools/timing.py 2 > gpurun_out/timing_c2.log 2>&1
cat gpurun_out/cta_c5.log; tail -3 gpurun_out/timing_c5.log; cat gpurun_out/timing_c2.log
