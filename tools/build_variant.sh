#!/bin/bash
# usage: tools/build_variant.sh NAME "-DFLAG=1 ..."  -> tools/variants/NAME.so (same flags as _build.py)
set -e
mkdir -p tools/variants
nvcc -gencode arch=compute_100a,code=sm_100a -O3 -lineinfo -std=c++17 -Xptxas -v -shared -Xcompiler -fPIC \
  --expt-relaxed-constexpr $2 -Iinclude paper_1702_07578_b200/csrc/wvlt_b200.cu -o tools/variants/$1.so -lcudart \
  > tools/variants/$1.log 2>&1 || { tail -20 tools/variants/$1.log; exit 1; }
grep -A3 "level_pass_u8_kernelILi4" tools/variants/$1.log | grep -E "registers|spill" | tr '\n' ' '; echo
