#!/bin/bash
# usage: scripts/sass_stats.sh <file.cu> <kernel-name-regex>   -> regs/spills + SASS opcode histogram
set -e
ROOT=/root/repo
SRC=$1; PAT=$2
/usr/local/cuda/bin/nvcc -gencode arch=compute_100a,code=sm_100a -O3 -std=c++17 --expt-relaxed-constexpr \
  -I$ROOT/include -I$ROOT/paper_2309_16849_b200/csrc -Xptxas -v -cubin -o /tmp/sass_stats.cubin $SRC 2>&1 \
  | grep -A2 -E "Compiling entry.*$PAT" | grep -E "Used|spill" | head -4
cuobjdump -sass /tmp/sass_stats.cubin | awk -v pat="$PAT" '/Function : /{f = ($0 ~ pat)} f' > /tmp/sass_stats.sass
echo "instructions: $(grep -cE '^\s+/\*[0-9a-f]{4}\*/' /tmp/sass_stats.sass)"
grep -oE '^\s+/\*[0-9a-f]{4}\*/\s+(@!?U?P[0-9T] )?[A-Z0-9]+' /tmp/sass_stats.sass | awk '{print $NF}' | sort | uniq -c | sort -rn | head -${3:-15} | tr '\n' ' '; echo
