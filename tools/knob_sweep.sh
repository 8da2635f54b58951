# plan-knob sweep on C3 and C5 (1 GiB): ring depth, static share, pool share
mkdir -p gpurun_out
{
for o in "" "ring_slots=3" "ctg64=32" "ctg64=56" "ctg64=60" "pool64=2" "pool64=8" "pool64=0"; do
  echo "== C3 $o"; python tools/qt.py 3:1024 $o 2>&1 | tail -1
done
for o in "" "ring_slots=3" "ctg64=32" "ctg64=56" "ctg64=60" "pool64=2" "pool64=8" "placement=global"; do
  echo "== C5 $o"; python tools/qt.py 5:1024 $o 2>&1 | tail -1
done
} > gpurun_out/knobs.log 2>&1
