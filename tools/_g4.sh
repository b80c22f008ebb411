./tools/ubench_tma > gpurun_out/ubench_tma.log 2>&1; cat gpurun_out/ubench_tma.log
python -m pytest tests/test_gpu_variants.py -x -q -k dstep > gpurun_out/t_dstep.log 2>&1; tail -2 gpurun_out/t_dstep.log
