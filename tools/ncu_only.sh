# plain run then one ncu --set full capture of the scan kernel (C2 bench step)
mkdir -p gpurun_out
python bench.py --steps 5 --warmup 3 --no-e2e --no-cpu-baseline > gpurun_out/plain.log 2>&1 && \
ncu --set full --clock-control none --import-source on -k regex:pfac_scan -s 4 -c 1 -o gpurun_out/prof python bench.py --steps 5 --warmup 3 --no-e2e --no-cpu-baseline > gpurun_out/ncu2.log 2>&1; echo ncu rc=$?
