# ncu --set full of the scan kernel on config ${CFG:-3} (tools/timing.py; plain run first)
mkdir -p gpurun_out
c=${CFG:-3}
export PFAC_LIB=${PFAC_LIB:-paper_1702_03657_b200/libpfac_timing.so}
python tools/timing.py $c > gpurun_out/plain_c$c.log 2>&1 && \
ncu --set full --clock-control none --import-source on -k regex:pfac_scan -s 1 -c 1 -o gpurun_out/prof_c$c python tools/timing.py $c > gpurun_out/ncu_c$c.log 2>&1; echo ncu rc=$?
