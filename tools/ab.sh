# A/B env variants on the default bench (per-kernel ms of the step)
for v in "GQ_X=0" "GQ_CHAIN_P=3" "GQ_X=0"; do
  env $v python bench.py --steps 30 --warmup 3 --no-cpu-baseline 2>/dev/null | python -c "import json,sys; d=json.load(sys.stdin); k=d['kernel_ms']; print('$v', round(d['value'],1), k['sweep_s0_l0'], k['sweep_s0_l1'], k['sweep_s1_l0'], k['sweep_s1_l1'])"
done
