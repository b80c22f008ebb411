for c in 1 2 3; do
timeout 300 python bench.py --config $c --steps 200 --warmup 10 --no-cpu-baseline > gpurun_out/c$c.json 2> gpurun_out/c$c.err; tail -2 gpurun_out/c$c.err
python -c "import json; d=json.loads(open('gpurun_out/c$c.json').read().strip().splitlines()[-1]); print($c, d['value'], d['ms_per_step'], d['kernel_ms'])"
done
