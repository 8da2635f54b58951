# ncu --set full of the production scan kernel on config ${CFG:-4} (1 GiB; plain run first)
mkdir -p gpurun_out
c=${CFG:-4}
python tools/plan.py $c > gpurun_out/plain_c$c.log 2>&1 && \
ncu --set full --clock-control none --import-source on -k regex:pfac_scan -c 1 -o gpurun_out/prof_c$c python tools/plan.py $c > gpurun_out/ncu_c$c.log 2>&1; echo ncu rc=$?
