mkdir -p gpurun_out
export CTSM_BENCH_NO_CPU=1
python bench.py --steps 1 --warmup 1 --no-e2e --no-clocks > gpurun_out/plain.log 2>&1 && \
ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches_r1a.csv python bench.py --steps 1 --warmup 1 --no-e2e --no-clocks > gpurun_out/ncu_launch.log 2>&1
ncu --set full --clock-control none --import-source on -k regex:"fwd2d|bwd2d" -s 2 -c 2 -o gpurun_out/prof_r1a python bench.py --steps 1 --warmup 1 --no-e2e --no-clocks > gpurun_out/ncu_full.log 2>&1
tail -3 gpurun_out/ncu_full.log
