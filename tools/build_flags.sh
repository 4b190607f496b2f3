#!/bin/bash
# Build the working tree's libprnet with extra nvcc flags into paper_2404_02445_b200/<NAME>
# (A/B experiments: PRNET_LIB=$PWD/paper_2404_02445_b200/<NAME> python bench.py ...).
set -eu
NAME=$1; shift
ROOT=$(cd "$(dirname "$0")/.." && pwd)
/usr/local/cuda/bin/nvcc -gencode arch=compute_100a,code=sm_100a -O3 -lineinfo -std=c++17 -shared \
  -Xcompiler -fPIC -I "$ROOT/include" "$@" -o "$ROOT/paper_2404_02445_b200/$NAME" "$ROOT"/paper_2404_02445_b200/csrc/*.cu
echo "built $NAME $*"
