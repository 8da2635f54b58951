# round-2 measurement batch: full GPU suite, bench line, ncu launch list, ncu --set full of the C4 4 GiB launch
mkdir -p gpurun_out
timeout 1500 python -m pytest tests -m gpu -q > gpurun_out/gputest_r02.log 2>&1; echo "rc=$?" >> gpurun_out/gputest_r02.log
python bench.py --steps 10 --warmup 3 > gpurun_out/bench_r02.json 2> gpurun_out/bench_r02.err
ncu --metrics gpu__time_duration.sum --clock-control none -k regex:pfac_scan --csv --log-file gpurun_out/launches_r02.csv \
    python bench.py --steps 2 --warmup 1 --no-e2e --no-cpu-baseline --no-verify --no-extras > gpurun_out/ncu_list.log 2>&1
python tools/run_cfg.py 4 4096 2 > gpurun_out/plain_c4full.log 2>&1 && \
ncu --set full --clock-control none --import-source on -k regex:pfac_scan -s 1 -c 1 -o gpurun_out/prof_c4full \
    python tools/run_cfg.py 4 4096 2 > gpurun_out/ncu_c4full.log 2>&1; echo "ncu rc=$?" >> gpurun_out/ncu_c4full.log
