#!/bin/bash
# pageable-numpy upload rate vs the staging chunk size (KSVD_IO_CHUNK_BYTES) and io threads
cd "${GRAFT_REPO_ROOT:-.}"
for cb in 8388608 16777216 33554432 67108864; do
  for th in 8 12; do
    echo "chunk $cb threads $th"; KSVD_IO_THREADS=$th KSVD_IO_CHUNK_BYTES=$cb timeout 300 python tools/upload_bench.py 2>&1 | sed -n 2,3p
  done
done
