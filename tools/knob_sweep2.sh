mkdir -p gpurun_out
{
for o in "" "ctg64=56" "ctg64=60" "ctg64=56 pool64=2" "ctg64=60 pool64=2" ""; do
  echo "== C5 $o"; python tools/qt.py 5:2048 $o 2>&1 | tail -1
done
for o in "" "pool64=2" "pool64=3" ""; do
  echo "== C3 $o"; python tools/qt.py 3:1024 $o 2>&1 | tail -1
done
} > gpurun_out/knobs2.log 2>&1
