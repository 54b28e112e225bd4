timeout 1500 python -m pytest tests -m gpu -q -x -p no:cacheprovider -k "parity or host_calls" 2>&1 | tail -4
python bench.py --gpus 1 --steps 10 --warmup 3 --no-cpu 2>&1 | tail -1 | cut -c1-900
CTSM_NO_PLAN_PASS=1 python bench.py --gpus 1 --steps 10 --warmup 3 --no-cpu 2>&1 | tail -1 | cut -c1-300
python bench.py --config c4 --mode sirt --steps 2 --warmup 1 --no-cpu 2>&1 | tail -1 | cut -c1-300
