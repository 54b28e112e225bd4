IFS='|' read -ra VS <<< "${VARIANTS}"
for v in "${VS[@]}"; do
  CTSM_NVCC_EXTRA="$v" python -c "from paper_2511_12235_b200 import build as b; b.build(force=True)" > /dev/null 2>&1 || { echo "build failed: $v"; continue; }
  echo "== [$v] $(python bench.py --mode csr --config c2 --steps 1 --warmup 2 --no-clocks 2>&1 | tail -1 | cut -c1-330)"
done
python -c "from paper_2511_12235_b200 import build as b; b.build(force=True)" > /dev/null 2>&1
