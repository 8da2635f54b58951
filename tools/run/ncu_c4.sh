python tools/run_cfg.py 4 256 2 > gpurun_out/plain_c4.log 2>&1 && \
ncu --set full --clock-control none --import-source on -k regex:pfac_scan -s 1 -c 1 -o gpurun_out/prof_c4 python tools/run_cfg.py 4 256 2 > gpurun_out/ncu_c4.log 2>&1; echo ncu rc=$?
python tools/run_cfg.py 5 256 2 > gpurun_out/plain_c5.log 2>&1 && \
ncu --set full --clock-control none --import-source on -k regex:pfac_scan -s 1 -c 1 -o gpurun_out/prof_c5 python tools/run_cfg.py 5 256 2 > gpurun_out/ncu_c5.log 2>&1; echo ncu rc=$?
