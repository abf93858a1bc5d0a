# A/B: base (build/libcw_base.so) vs working tree (in-tree .so), alternating
for i in 1 2; do
 CW_B200_LIB=build/libcw_base.so python bench.py --steps 1500 --warmup 20 --no-cpu-baseline > gpurun_out/base$i.json 2>/dev/null
 python bench.py --steps 1500 --warmup 20 --no-cpu-baseline > gpurun_out/new$i.json 2>/dev/null
done
python - <<'PY'
import json
for f in ("base1","new1","base2","new2"):
    d=json.loads(open(f"gpurun_out/{f}.json").read().strip().splitlines()[-1])
    print(f, round(d["ms_per_step"],4), round(d["roofline"]["frac"],4), "kernel_ms", round(d["roofline"].get("kernel_ms",0),4), "e2e", round(d["e2e"]["value"]/1e9,3))
PY
