for v in "GQ_GRID2=0" "GQ_GRID2_STRIPS=1" "GQ_GRID2_STRIPS=2" "GQ_GRID2_STRIPS=3" "GQ_GRID2_STRIPS=4"; do
  env $v python bench.py --steps 30 --warmup 3 --no-cpu-baseline 2>/dev/null | python -c "import json,sys; d=json.load(sys.stdin); k=d['kernel_ms']; print('$v', round(d['value'],1), k['delta'], k['outer_rhs_s1'])"
done
