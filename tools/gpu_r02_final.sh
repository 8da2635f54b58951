# round-2 final batch: GPU suite, checked-build suite, bench line, ncu launch list + full capture of the C4 4 GiB launch, C3/C5 captures, placement table
mkdir -p gpurun_out
timeout 1800 python -m pytest tests -m gpu -q > gpurun_out/gputest_final.log 2>&1; echo "rc=$?" >> gpurun_out/gputest_final.log
bash tools/checked_tests.sh
python bench.py --steps 10 --warmup 3 > gpurun_out/bench_final.json 2> gpurun_out/bench_final.err
python bench.py --impl reference --steps 3 --warmup 1 > gpurun_out/bench_ref.json 2> gpurun_out/bench_ref.err
ncu --metrics gpu__time_duration.sum --clock-control none -k regex:pfac_scan --csv --log-file gpurun_out/launches_final.csv \
    python bench.py --steps 2 --warmup 1 --no-e2e --no-cpu-baseline --no-verify --no-extras > gpurun_out/ncu_list.log 2>&1
python tools/run_cfg.py 4 4096 2 > gpurun_out/plain_c4full.log 2>&1 && \
ncu --set full --clock-control none --import-source on -k regex:pfac_scan -s 1 -c 1 -o gpurun_out/prof_c4final \
    python tools/run_cfg.py 4 4096 2 > gpurun_out/ncu_c4final.log 2>&1
for c in 3 5; do
python tools/run_cfg.py $c 256 2 > gpurun_out/plain_c$c.log 2>&1 && \
ncu --set full --clock-control none --import-source on -k regex:pfac_scan -s 1 -c 1 -o gpurun_out/prof_c${c}final \
    python tools/run_cfg.py $c 256 2 > gpurun_out/ncu_c${c}final.log 2>&1
done
timeout 900 python tools/placement.py 2 3 4 5 > gpurun_out/placement_final.jsonl 2>&1
