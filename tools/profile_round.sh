mkdir -p gpurun_out/r02d
python bench.py > gpurun_out/r02d/bench_default.json 2> gpurun_out/r02d/bench_default.err; tail -2 gpurun_out/r02d/bench_default.err
python bench.py --steps 2 --warmup 1 --no-cpu-baseline > gpurun_out/r02d/plain.log 2>&1 && \
ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/r02d/launches_bench_steps2.csv python bench.py --steps 2 --warmup 1 --no-cpu-baseline > gpurun_out/r02d/ncu_launch.log 2>&1
bash tools/ncu_step.sh step_r02d
python tools/configs_report.py > gpurun_out/r02d/configs.json 2> gpurun_out/r02d/configs.err; tail -2 gpurun_out/r02d/configs.err
