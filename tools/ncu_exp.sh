# ncu --set full of the scan kernel in the production build (bench workload) and
# in the filter-only experiment build (tools/timing.py C2); plain runs first
mkdir -p gpurun_out
bash tools/ncu_only.sh
PFAC_LIB=paper_1702_03657_b200/libpfac_exp1.so python tools/timing.py 2 > gpurun_out/plain_exp1.log 2>&1 && \
PFAC_LIB=paper_1702_03657_b200/libpfac_exp1.so ncu --set full --clock-control none --import-source on -k regex:pfac_scan -s 2 -c 1 -o gpurun_out/prof_exp1 python tools/timing.py 2 > gpurun_out/ncu_exp1.log 2>&1; echo ncu exp1 rc=$?
