mkdir -p gpurun_out
{
for o in "" "pool64=2" "pool64=1" "pool64=8" "pool64=0" ""; do
  echo "== C4 $o"; python tools/qt.py 4:4096 $o 2>&1 | tail -1
done
for o in "" "ctg64=40" "ctg64=44" "ctg64=52" ""; do
  echo "== C3 $o"; python tools/qt.py 3:1024 $o 2>&1 | tail -1
done
} > gpurun_out/knobs3.log 2>&1
