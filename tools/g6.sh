export GQ_CHAINX=1
timeout 600 python -m pytest tests/test_gpu_parity.py -m gpu -x -q 2>&1 | tail -2
for v in "8 10" "6 10" "4 7"; do set -- $v
GQ_CHAINX_PI=$1 GQ_CHAINX_PO=$2 timeout 300 python bench.py --steps 50 --warmup 5 --no-cpu-baseline > gpurun_out/bx.json 2>/dev/null
python -c "import json; d=json.loads(open('gpurun_out/bx.json').read().strip().splitlines()[-1]); print('$v', round(d['value'],1), d['kernel_ms'])"
done
GQ_CHAINX=0 timeout 300 python bench.py --steps 50 --warmup 5 --no-cpu-baseline > gpurun_out/bx.json 2>/dev/null
python -c "import json; d=json.loads(open('gpurun_out/bx.json').read().strip().splitlines()[-1]); print('base', round(d['value'],1), d['kernel_ms'])"
