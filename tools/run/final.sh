NCU=1 bash tools/gpu_round.sh
timeout 900 python tools/config_table.py > gpurun_out/config_table.jsonl 2> gpurun_out/config_table.err; echo cfg rc=$?
timeout 600 python bench.py --impl reference > gpurun_out/ref.json 2> gpurun_out/ref.err; echo ref rc=$?
