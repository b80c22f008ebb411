python -m pytest tests/test_gpu_parity.py tests/test_gpu_variants.py -x -q > gpurun_out/t5.log 2>&1; tail -3 gpurun_out/t5.log
for v in "" "GQ_NO_ORHS=1" ""; do
  env $v python bench.py --steps 100 --warmup 5 --no-cpu-baseline > gpurun_out/b5_${v%%=*}.json 2>gpurun_out/b5.err
  python -c "
import json; d=json.loads(open('gpurun_out/b5_${v%%=*}.json').read().strip().splitlines()[-1]); print('$v', round(d['value'],1), round(d['e2e']['value'],1), {k:round(x,4) for k,x in d['kernel_ms'].items()})"
done
bash tools/ncu_kernel.sh k_orhs orhs3 1
