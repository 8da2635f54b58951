# compute-sanitizer runs (profiles/r02/sanitizer_*.log) + the placement ablation
mkdir -p gpurun_out
CS=/usr/local/cuda/bin/compute-sanitizer
python tools/san_run.py > gpurun_out/san_plain.log 2>&1; echo "plain rc=$?" >> gpurun_out/san_plain.log
timeout 1500 $CS --tool memcheck --leak-check full --error-exitcode 9 python tools/san_run.py > gpurun_out/sanitizer_memcheck.log 2>&1; echo "rc=$?" >> gpurun_out/sanitizer_memcheck.log
SAN_MIB=1 timeout 2400 $CS --tool racecheck --racecheck-report all --error-exitcode 9 python tools/san_run.py > gpurun_out/sanitizer_racecheck.log 2>&1; echo "rc=$?" >> gpurun_out/sanitizer_racecheck.log
timeout 1500 $CS --tool synccheck --error-exitcode 9 python tools/san_run.py > gpurun_out/sanitizer_synccheck.log 2>&1; echo "rc=$?" >> gpurun_out/sanitizer_synccheck.log
python tools/placement.py 2 3 4 5 > gpurun_out/placement_r02.jsonl 2>&1
