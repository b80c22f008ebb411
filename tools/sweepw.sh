for cfg in "0 1 2" "1 1 1" "1 1 2" "1 1 3" "1 2 1" "1 2 2"; do
  set -- $cfg
  GQ_CHAIN_X=$1 GQ_CHAIN_MT=$2 GQ_CHAINX_P=$3 python bench.py --steps 20 --warmup 3 --no-cpu-baseline 2>/dev/null | python -c "import json,sys; d=json.load(sys.stdin); k=d['kernel_ms']; print('X=$1 MT=$2 P=$3', round(d['value'],1), k['sweep_s0_l0'], k['sweep_s0_l1'], k['sweep_s1_l1'])"
done
