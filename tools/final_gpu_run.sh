# Round-end measurement set on one B200 (outputs under gpurun_out/):
# GPU tests, smoke, headline bench, reference arm, other configs, ncu launch
# list and one full ncu capture of the frame kernel.
set -x
python -m pytest tests -m gpu -x -q > gpurun_out/pytest_gpu.log 2>&1
python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke.log 2>&1
python bench.py > gpurun_out/bench_c3.json 2> gpurun_out/bench_c3.err
python bench.py --impl reference --steps 3 --warmup 3 > gpurun_out/bench_ref.json 2> gpurun_out/bench_ref.err
for c in c2 c4 c5 c3naive c3seq; do
  python bench.py --config $c --no-cpu-baseline > gpurun_out/bench_$c.jsonl 2> gpurun_out/bench_$c.err
done
ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches.csv \
  python bench.py --steps 60 --warmup 5 --no-cpu-baseline > gpurun_out/ncu_launch.log 2>&1
ncu --set full --clock-control none --import-source on -k regex:cw_frame_kernel -s 8 -c 1 -f \
  -o gpurun_out/final python tools/prof_frame.py 12 > gpurun_out/ncu_full.log 2>&1
tail -2 gpurun_out/pytest_gpu.log; cat gpurun_out/smoke.log gpurun_out/bench_c3.json
