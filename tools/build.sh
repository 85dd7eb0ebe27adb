#!/bin/bash
# dev build with ptxas report: tools/build.sh [filter]
cd "$(dirname "$0")/.." || exit 1
nvcc -gencode arch=compute_100a,code=sm_100a -O3 -lineinfo -std=c++17 -Xptxas -v -shared -Xcompiler -fPIC \
  -o paper_1808_00896_b200/libso3fft_b200.so paper_1808_00896_b200/csrc/so3fft_b200.cu > /tmp/build.log 2>&1
rc=$?
grep -E "error" /tmp/build.log | head -20
grep -A3 "Compiling entry" /tmp/build.log | grep -E "Compiling|registers|spill" | sed -E 's/ptxas info *: //' | paste - - - | grep -E "${1:-.}" | awk '{print substr($0,1,230)}'
exit $rc
