# one GPU round: smoke, gpu tests, bench, ncu launch list + full capture of the scan kernel
set -x
mkdir -p gpurun_out
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm,clocks.mem --format=csv
python __graft_entry__.py smoke > gpurun_out/smoke.log 2>&1; echo smoke rc=$?
timeout 900 python -m pytest tests -m gpu -x -q > gpurun_out/gpu_tests.log 2>&1; echo tests rc=$?
python bench.py > gpurun_out/bench.json 2> gpurun_out/bench.err; echo bench rc=$?
if [ "${NCU:-1}" = "1" ]; then
python bench.py --steps 5 --warmup 3 --no-e2e --no-cpu-baseline > gpurun_out/plain.log 2>&1 && \
ncu --metrics gpu__time_duration.sum --clock-control none -c 60 --csv --log-file gpurun_out/launches.csv python bench.py --steps 5 --warmup 3 --no-e2e --no-cpu-baseline > gpurun_out/ncu1.log 2>&1 && \
ncu --set full --clock-control none --import-source on -k regex:pfac_scan -s 4 -c 1 -o gpurun_out/prof python bench.py --steps 5 --warmup 3 --no-e2e --no-cpu-baseline > gpurun_out/ncu2.log 2>&1; echo ncu rc=$?
fi
