make -s paper_1702_03657_b200/libpfac_timing.so
for c in 64 60 48; do PFAC_CTG64=$c PFAC_LIB=paper_1702_03657_b200/libpfac_timing.so timeout 300 python tools/timing.py 2 > gpurun_out/timing_c2_$c.log 2>&1; echo "== $c"; grep -E "phase1 end|offsets known|^end|local scan|per-CTA|duration" gpurun_out/timing_c2_$c.log; done
