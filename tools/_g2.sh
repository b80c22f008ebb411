GQ_DSTEP=1 timeout 300 compute-sanitizer --tool memcheck python tools/_dbg.py boundary > gpurun_out/san.log 2>&1; head -60 gpurun_out/san.log
GQ_DSTEP=1 timeout 300 python tools/_dbg.py config1 config2 odd_kn time_varying config4r sparse > gpurun_out/dbg2.log 2>&1; cat gpurun_out/dbg2.log | tail -20
bash tools/ncu_kernel.sh k_orhs orhs1 1
