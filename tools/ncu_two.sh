# ncu --set full captures of the scan on C4 (1 GiB) and C5 (1 GiB) with the current build
mkdir -p gpurun_out
for c in 4 5; do
python tools/run_cfg.py $c 1024 2 > gpurun_out/plain_c$c.log 2>&1 && \
ncu --set full --clock-control none --import-source on -k regex:pfac_scan -s 1 -c 1 -o gpurun_out/prof_c${c}_cur \
    python tools/run_cfg.py $c 1024 2 > gpurun_out/ncu_c${c}_cur.log 2>&1; echo "c$c ncu rc=$?"
done
