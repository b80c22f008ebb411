GQ_DSTEP=1 timeout 600 python -m pytest tests/test_gpu_parity.py -m gpu -x -q -k "unit_applies or pcg_parity" 2>&1 | tail -2
timeout 600 python -m pytest tests/test_gpu_parity.py -m gpu -x -q -k "full_size or headline" 2>&1 | tail -2
timeout 300 python bench.py --steps 50 --warmup 5 --no-cpu-baseline > gpurun_out/b14.json 2> gpurun_out/b14.err; tail -2 gpurun_out/b14.err
python -c "import json; d=json.loads(open('gpurun_out/b14.json').read().strip().splitlines()[-1]); print(d['value'], d['e2e']['value'], d['kernel_ms'])"
bash tools/ncu_kernel.sh k_dstep dstep12 1
