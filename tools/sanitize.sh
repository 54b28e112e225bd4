#!/bin/bash
# compute-sanitizer over the small-geometry tour, one tool per call
# (SURVEY.md §5). Usage: TOOL=memcheck TAG=r2 bash tools/sanitize.sh
TOOL=${TOOL:-memcheck}
TAG=${TAG:-r2}
mkdir -p gpurun_out
python tools/sanitize_driver.py > gpurun_out/${TAG}_sanitize_plain.log 2>&1 || { tail -5 gpurun_out/${TAG}_sanitize_plain.log; exit 1; }
timeout 2400 compute-sanitizer --tool ${TOOL} --error-exitcode 3 --print-limit 20 \
  python tools/sanitize_driver.py > gpurun_out/${TAG}_sanitize_${TOOL}.log 2>&1
echo "exit $?" >> gpurun_out/${TAG}_sanitize_${TOOL}.log
tail -6 gpurun_out/${TAG}_sanitize_${TOOL}.log
