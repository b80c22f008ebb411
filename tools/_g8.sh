python bench.py --steps 100 --warmup 5 --no-cpu-baseline > gpurun_out/b8.json 2>gpurun_out/b8.err
python -c "
import json; d=json.loads(open('gpurun_out/b8.json').read().strip().splitlines()[-1]); print(round(d['value'],1), round(d['e2e']['value'],1), {k:round(x,4) for k,x in d['kernel_ms'].items()})"
for c in 1 2; do
ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launch_c$c.csv python bench.py --config $c --steps 3 --warmup 3 --no-cpu-baseline > /dev/null 2>&1
done
ls -la gpurun_out/launch_c*.csv
