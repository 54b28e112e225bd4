#!/bin/bash
# ncu launch list and one full capture of the dominant kernels of the DEFAULT
# bench command (B200_PROFILING.md recipe): the same command first without ncu.
# Usage: TAG=r2t bash tools/ncu_bench.sh
TAG=${TAG:-r2t}
mkdir -p gpurun_out
ARGS="--gpus 1 --steps 2 --warmup 1 --no-cpu --no-e2e --no-clocks"
python bench.py $ARGS > gpurun_out/${TAG}_bench_plain.json 2> gpurun_out/${TAG}_bench_plain.err || exit 1
ncu --metrics gpu__time_duration.sum --clock-control none -c 600 --csv \
  --log-file gpurun_out/${TAG}_bench_launches.csv python bench.py $ARGS > /dev/null 2>&1
ncu --set full --clock-control none --import-source on -k regex:"fwd3d_sym|bwd3d_sym" -s 2 -c 2 -f \
  -o gpurun_out/${TAG}_bench_3d python bench.py $ARGS > /dev/null 2>&1
ls -la gpurun_out | grep ${TAG}
