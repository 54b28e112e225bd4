#!/bin/bash
# ncu of the 2D matrix-free kernels on C1 (one timed step).
mkdir -p gpurun_out
export CTSM_BENCH_NO_CPU=1
TAG=${TAG:-r1c}
python bench.py --steps 1 --warmup 1 --no-e2e --no-clocks > gpurun_out/plain_${TAG}.log 2>&1 && \
ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches_${TAG}.csv python bench.py --steps 1 --warmup 1 --no-e2e --no-clocks > gpurun_out/ncu_launch_${TAG}.log 2>&1
ncu --set full --clock-control none --import-source on -k regex:"fwd2d|bwd2d" -s 2 -c 2 -o gpurun_out/prof_${TAG} python bench.py --steps 1 --warmup 1 --no-e2e --no-clocks > gpurun_out/ncu_full_${TAG}.log 2>&1
tail -2 gpurun_out/ncu_full_${TAG}.log
