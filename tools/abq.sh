# A/B of library builds on one config (alternating processes): bash tools/abq.sh CFG:MiB lib1 lib2 ...
c=$1; shift
for rep in 1 2; do for lib in "$@"; do
  echo -n "$lib "; PFAC_LIB=$PWD/paper_1702_03657_b200/$lib python tools/qt.py $c 2>&1 | tail -1
done; done
