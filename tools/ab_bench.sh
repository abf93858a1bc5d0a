# A/B/...: alternating 1-GPU benches of several builds of the library.
# usage: bash tools/ab_bench.sh [lib ...]   (default: build/libcw_base.so and the in-tree build)
libs=("$@")
[ ${#libs[@]} -eq 0 ] && libs=(build/libcw_base.so paper_1408_3526_b200/libcw_b200.so)
for i in 1 2; do
  for l in "${libs[@]}"; do
    n=$(basename "$l" .so)
    CW_B200_LIB=$l python bench.py --steps 1500 --warmup 20 --no-cpu-baseline > gpurun_out/ab_${n}_$i.json 2>/dev/null
  done
done
python - "${libs[@]}" <<'PY'
import json, os, sys
for i in (1, 2):
    for l in sys.argv[1:]:
        n = os.path.basename(l)[:-3]
        try:
            d = json.loads(open(f"gpurun_out/ab_{n}_{i}.json").read().strip().splitlines()[-1])
            print(f"{n:24s} run{i} step_ms {d['ms_per_step']:.4f} frac {d['roofline']['frac']:.4f} kernel_ms {d['roofline'].get('kernel_ms', 0):.4f}")
        except Exception as e:
            print(n, i, "failed", e)
PY
