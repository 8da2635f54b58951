mkdir -p gpurun_out
{
for o in "" "stage2=0" "placement=smem hot_bytes_cap=8192" "placement=smem hot_bytes_cap=32768" "placement=global max_filter_rep_log2=0" "placement=global max_filter_rep_log2=1 ring_slots=2" ""; do
  echo "== C3 $o"; python tools/qt.py 3:1024 $o 2>&1 | tail -1
done
} > gpurun_out/knobs4.log 2>&1
