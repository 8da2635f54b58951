# ncu capture of the scan on config $1 ($2 MiB): plain run first, then ncu
mkdir -p gpurun_out
python tools/run_cfg.py $1 $2 2 > gpurun_out/plain_cfg.log 2>&1 && \
ncu --set full --clock-control none --import-source on -k regex:pfac_scan -s 1 -c 1 -o gpurun_out/prof_c$1 python tools/run_cfg.py $1 $2 2 > gpurun_out/ncu_cfg.log 2>&1; echo ncu rc=$?
