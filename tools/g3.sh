
timeout 600 python -m pytest tests/test_gpu_parity.py tests/test_gpu_edges.py -m gpu -x -q 2>&1 | tail -3
timeout 300 python bench.py --steps 50 --warmup 5 --no-cpu-baseline > gpurun_out/b13.json 2> gpurun_out/b13.err; tail -3 gpurun_out/b13.err
python -c "import json; d=json.loads(open('gpurun_out/b13.json').read().strip().splitlines()[-1]); print(d['value'], d['e2e']['value'], d['kernel_ms'])"
bash tools/ncu_kernel.sh k_chainx chx2 4
