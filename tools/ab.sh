for i in 1 2; do
  python bench.py --steps 30 --warmup 3 --no-cpu-baseline 2>/dev/null | python -c "import json,sys; d=json.load(sys.stdin); k=d['kernel_ms']; print(round(d['value'],1), k['delta'], k['outer_rhs_s1'])"
done
