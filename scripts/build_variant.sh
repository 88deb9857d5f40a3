#!/bin/bash
# A/B helper: build a copy of libsnls_cuda.so with search_tiled.cu compiled under extra
# defines, for bench runs with SNLS_LIB_OVERRIDE=<out>.
# usage: scripts/build_variant.sh OUT.so -DSNLS_X=0 ...
set -e
out=$1; shift
root=$(cd "$(dirname "$0")/.." && pwd)
pkg=$root/paper_2309_16849_b200
python -c "import sys; sys.path.insert(0, '$root'); from paper_2309_16849_b200 import build; build.build()"
tmp=$(mktemp -d)
/usr/local/cuda/bin/nvcc -gencode arch=compute_100a,code=sm_100a -O3 -lineinfo -std=c++17 -Xcompiler -fPIC \
  --expt-relaxed-constexpr -I "$root/include" -I "$pkg/csrc" "$@" -c "${SRC:-$pkg/csrc/${UNIT:-search_tiled}.cu}" -o "$tmp/${UNIT:-search_tiled}.o"
objs=$(ls "$pkg"/build/*.o | grep -v ${UNIT:-search_tiled}.o)
/usr/local/cuda/bin/nvcc -gencode arch=compute_100a,code=sm_100a -shared -o "$out" $objs "$tmp/${UNIT:-search_tiled}.o" -cudart static -ldl
rm -rf "$tmp"
