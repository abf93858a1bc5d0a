#!/bin/bash
# Fast dev build: only the default geometry (4,4,2,3,3) with 17 lags (+ the
# runtime-loop instance).  Output: $1 (default build/libcw_dev.so); use with
# CW_B200_LIB=... .  Prints the frame kernels' register / spill report.
set -e
cd "$(dirname "$0")/.."
out=${1:-build/libcw_dev.so}
shift || true
nvcc -gencode arch=compute_100a,code=sm_100a -O3 -lineinfo -std=c++17 -Xcompiler -fPIC -shared \
  -DCW_DEV_DEFAULT_ONLY -Xptxas -v "$@" -o "$out" paper_1408_3526_b200/csrc/cw_api.cu 2>&1 |
  grep -A3 "Compiling entry.*cw_frame" | grep -o "Li[0-9]*EEEvNS_9Frame\|Used [0-9]* registers\|[0-9]* bytes spill stores" | paste -sd' '
