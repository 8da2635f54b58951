# parity + bench + per-phase timings (instrumented and experiment builds); no profiler
mkdir -p gpurun_out
timeout 900 python -m pytest tests -m gpu -x -q > gpurun_out/gpu_tests.log 2>&1; echo tests rc=$?
tail -2 gpurun_out/gpu_tests.log
python bench.py --no-cpu-baseline > gpurun_out/bench.json 2> gpurun_out/bench.err; echo bench rc=$?
for c in ${CFGS:-2 3 4 5}; do PFAC_LIB=paper_1702_03657_b200/libpfac_timing.so timeout 300 python tools/timing.py $c > gpurun_out/timing_c$c.log 2>&1; done
for e in exp1 exp2 stream; do PFAC_LIB=paper_1702_03657_b200/libpfac_$e.so timeout 300 python tools/timing.py 2 > gpurun_out/timing_$e.log 2>&1; done
