#!/bin/bash
# Static SASS opcode counts of one kernel instantiation (no GPU needed).
#   tools/sass_count.sh [cu-file] [kernel-regex]
# Default: the Traffic instantiation of the default kernel.
set -e
F=${1:-paper_2404_02445_b200/csrc/fwd_mma.cu}
K=${2:-'prnet_fwd_mma_kernelILi2ELi2ELi24ELb0ELi30E'}
D=$(mktemp -d)
nvcc -gencode arch=compute_100a,code=sm_100a -O3 -std=c++17 -cubin -Iinclude -Ipaper_2404_02445_b200/csrc \
  -Xptxas -v -o $D/k.cubin "$F" 2>$D/ptxas.txt
grep -A1 "$K" $D/ptxas.txt | grep -E "registers|spill" | head -3 || true
cuobjdump -sass $D/k.cubin | awk -v k="$K" '/Function :/{on = ($0 ~ k)} on' > $D/k.sass
grep -E '^\s+/\*[0-9a-f]{4}\*/' $D/k.sass | sed -E 's/^\s+\/\*[0-9a-f]+\*\/\s+//; s/^@!?U?P[0-9T] //' | awk '{split($1,a,"."); print a[1]}' | sort | uniq -c | sort -rn | awk '{t+=$1; printf "%6d %s\n",$1,$2} END {printf "%6d TOTAL\n", t}' | head -${TOP:-40}
rm -rf $D
