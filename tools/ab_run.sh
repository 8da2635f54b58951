# A/B of libpfac_prev.so vs libpfac_new.so on C4/C3/C5/C2 (tools/abq.sh), then the GPU suite on the new build
mkdir -p gpurun_out
{ for c in ${AB_CFGS:-4:4096 3:1024 5:1024 2:64}; do echo "== $c"; bash tools/abq.sh $c libpfac_prev.so libpfac_new.so; done; } > gpurun_out/ab.log 2>&1
if [ -z "$AB_NO_TESTS" ]; then
timeout 1200 python -m pytest tests -m gpu -q -x > gpurun_out/gputest_ab.log 2>&1; echo "rc=$?" >> gpurun_out/gputest_ab.log
fi
