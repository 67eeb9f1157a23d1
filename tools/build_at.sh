#!/bin/bash
# Build libksvd.so as of git revision $1 into $2 (same-box A/B: KSVD_LIB_PATH=$2).
set -e
rev=$1; out=$2
tmp=$(mktemp -d)
git archive "$rev" paper_2104_10785_b200/csrc include paper_2104_10785_b200/build.py | tar -x -C "$tmp"
inc=$(python -c "import paper_2104_10785_b200.build as b; print(b._nccl_dirs()[0])")
lib=$(python -c "import paper_2104_10785_b200.build as b; print(b._nccl_dirs()[1])")
nvcc -gencode=arch=compute_100a,code=sm_100a -O3 -std=c++17 -lineinfo -shared \
  -Xcompiler -fPIC,-ffp-contract=off,-O3 -I"$tmp/include" -I"$tmp/paper_2104_10785_b200/csrc" -I"$inc" \
  "$tmp/paper_2104_10785_b200/csrc/ksvd.cu" "$tmp/paper_2104_10785_b200/csrc/eig.cpp" -o "$out" \
  -L"$lib" -l:libnccl.so.2 -lpthread -Xlinker=-rpath,"$lib"
rm -rf "$tmp"
echo "$out"
