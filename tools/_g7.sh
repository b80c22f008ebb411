GQ_DSTEP=1 python -m pytest tests/test_gpu_parity.py -x -q -k "unit or pcg_parity" > gpurun_out/t7.log 2>&1; tail -2 gpurun_out/t7.log
for v in "" "GQ_DSTEP_YTMA=1" ""; do
  env $v python bench.py --steps 100 --warmup 5 --no-cpu-baseline > gpurun_out/b7.json 2>gpurun_out/b7.err
  python -c "
import json; d=json.loads(open('gpurun_out/b7.json').read().strip().splitlines()[-1]); print('$v', round(d['value'],1), round(d['e2e']['value'],1), {k:round(x,4) for k,x in d['kernel_ms'].items()})"
done
