# Round-end measurement set on one B200 (outputs under gpurun_out/, prefix $P):
# headline bench, reference arm, other configs, ncu launch list and one
# full ncu capture of the frame kernel.
P=${1:-r02}
set -x
python bench.py > gpurun_out/${P}_bench_c3.json 2> gpurun_out/${P}_bench_c3.err
python bench.py --impl reference --steps 3000 --warmup 20 > gpurun_out/${P}_bench_ref.json 2> gpurun_out/${P}_bench_ref.err
for c in c2 c5 jit c4strips c3naive c3seq; do
  python bench.py --config $c --no-cpu-baseline --steps 1000 > gpurun_out/${P}_bench_$c.jsonl 2> gpurun_out/${P}_bench_$c.err
done
ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/${P}_launches.csv \
  python bench.py --steps 60 --warmup 5 --no-cpu-baseline --no-c4 > gpurun_out/${P}_ncu_launch.log 2>&1
ncu --set full --clock-control none --import-source on -k regex:cw_frame_kernel -s 8 -c 1 -f \
  -o gpurun_out/${P}_final python tools/prof_frame.py 12 > gpurun_out/${P}_ncu_full.log 2>&1
cat gpurun_out/${P}_bench_c3.json gpurun_out/${P}_bench_ref.json
