mkdir -p gpurun_out
{ for c in 4:4096 3:1024 5:1024 2:64; do echo "== $c"; bash tools/abq.sh $c libpfac_prev.so libpfac_new.so; done; } > gpurun_out/ab_smem.log 2>&1
timeout 1200 python -m pytest tests -m gpu -q -x > gpurun_out/gputest_smem.log 2>&1; echo "rc=$?" >> gpurun_out/gputest_smem.log
