# Build the scan library of git revision $1 (default HEAD) as
# paper_1702_03657_b200/libpfac_ref.so, for A/B timing against the working tree
# (tools/ab.py).  Sources are exported to .abtmp/ (git-ignored).
set -e
REV=${1:-HEAD}
rm -rf .abtmp && mkdir -p .abtmp/csrc .abtmp/include
for f in $(git ls-tree --name-only $REV paper_1702_03657_b200/csrc/); do git show $REV:$f > .abtmp/csrc/$(basename $f); done
git show $REV:include/pfac.h > .abtmp/include/pfac.h
/usr/local/cuda/bin/nvcc -O3 -lineinfo -std=c++17 -gencode arch=compute_100a,code=sm_100a -Xcompiler -fPIC,-Wall \
  -I.abtmp/include --expt-relaxed-constexpr -shared -o paper_1702_03657_b200/libpfac_ref.so \
  .abtmp/csrc/*.cu .abtmp/csrc/*.cpp -lcudart
echo built libpfac_ref.so from $REV
