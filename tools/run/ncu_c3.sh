python tools/run_cfg.py 3 256 2 > gpurun_out/plain_c3.log 2>&1 && \
ncu --set full --clock-control none --import-source on -k regex:pfac_scan -s 1 -c 1 -o gpurun_out/prof_c3 python tools/run_cfg.py 3 256 2 > gpurun_out/ncu_c3.log 2>&1; echo ncu rc=$?
