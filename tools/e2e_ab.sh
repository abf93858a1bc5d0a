# e2e probe (process_frame / cw_push host paths) for several library builds, alternating
for i in 1 2; do for l in "$@"; do echo "== $l"; CW_B200_LIB=$l python tools/e2e_probe.py 2>&1 | head -5; done; done
