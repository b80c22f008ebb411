for i in 1 2; do
for v in 0 1 2 3 4; do
  GQ_GRID_OCC=$v python bench.py --steps 30 --warmup 3 --no-cpu-baseline 2>/dev/null | python -c "import json,sys; d=json.load(sys.stdin); k=d['kernel_ms']; print('OCC=$v', round(d['value'],1), k['delta'])"
done; done
