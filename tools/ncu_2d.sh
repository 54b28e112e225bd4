#!/bin/bash
# ncu of the 2D matrix-free kernels on C1 (one timed step).
mkdir -p gpurun_out
TAG=${TAG:-r2o}
python bench.py --config c1 --steps 1 --warmup 1 --no-e2e --no-clocks --no-cpu > gpurun_out/plain_${TAG}.log 2>&1 && \
ncu --set full --clock-control none --import-source on -k regex:"fwd2d|bwd2d" -s 2 -c 2 -f -o gpurun_out/prof2d_${TAG} python bench.py --config c1 --steps 1 --warmup 1 --no-e2e --no-clocks --no-cpu > gpurun_out/ncu_full_${TAG}.log 2>&1
tail -2 gpurun_out/ncu_full_${TAG}.log
