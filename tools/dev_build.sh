#!/bin/bash
# Fast dev build: only the default geometry (4,4,2,3,3) with 17 and 33 lags (+ the
# runtime-loop instance).  Output: $1 (default build/libcw_dev.so); use with
# CW_B200_LIB=... .  Extra nvcc flags follow the output path.  Prints the
# frame kernels' register / spill report.
set -e
cd "$(dirname "$0")/.."
out=${1:-build/libcw_dev.so}
shift || true
python - "$out" "$@" <<'PY' 2>&1 | grep -A3 "Compiling entry.*cw_frame" | grep -o "Li[0-9]*EEEvNS_9Frame\|Used [0-9]* registers\|[0-9]* bytes spill stores" | paste -sd' '
import sys
sys.path.insert(0, ".")
from paper_1408_3526_b200 import _native
_native.build(verbose=True, out=sys.argv[1], dev=True, extra=sys.argv[2:])
PY
