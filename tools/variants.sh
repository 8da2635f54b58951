# A/B timing of layout variants (instrumented builds; no profiler)
mkdir -p gpurun_out
for v in timing v_s0 v_e0 v_s0e0; do for c in ${CFGS:-2 3}; do
  PFAC_LIB=paper_1702_03657_b200/libpfac_$v.so timeout 300 python tools/timing.py $c > gpurun_out/var_${v}_c$c.log 2>&1
done; done
