#!/bin/bash
# ncu of the 3D symmetric matrix-free kernels (C3 geometry, an orbit shard).
mkdir -p gpurun_out
TAG=${TAG:-r1d}
python tools/prof3d.py c3 64 > gpurun_out/prof3d_plain_${TAG}.log 2>&1 && \
ncu --set full --clock-control none --import-source on -k regex:"3d_sym" -s 2 -c 2 -f -o gpurun_out/prof3d_${TAG} python tools/prof3d.py c3 64 > gpurun_out/ncu3d_${TAG}.log 2>&1
tail -3 gpurun_out/prof3d_plain_${TAG}.log
