export STEPS=3
python tools/stepprof.py > gpurun_out/sp.log 2>&1 && \
ncu --set full --clock-control none --import-source on --launch-skip 13 -c 8 -o gpurun_out/step_r02a python tools/stepprof.py > gpurun_out/ncu_a.log 2>&1
tail -5 gpurun_out/ncu_a.log
