#!/bin/bash
# Build libprnet.so from git revision REV (default HEAD) into
# paper_2404_02445_b200/<OUT> (default libprnet_prev.so), for tools/ab.sh.
set -eu
REV=${1:-HEAD}
OUT=${2:-libprnet_prev.so}
ROOT=$(cd "$(dirname "$0")/.." && pwd)
TMP=$(mktemp -d)
git -C "$ROOT" archive "$REV" paper_2404_02445_b200/csrc include | tar -x -C "$TMP"
/usr/local/cuda/bin/nvcc -gencode arch=compute_100a,code=sm_100a -O3 -lineinfo -std=c++17 -shared \
  -Xcompiler -fPIC -I "$TMP/include" -o "$ROOT/paper_2404_02445_b200/$OUT" "$TMP"/paper_2404_02445_b200/csrc/*.cu
rm -rf "$TMP"
echo "built $REV -> paper_2404_02445_b200/$OUT"
