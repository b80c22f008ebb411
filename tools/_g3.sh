for T in 3 6 7 8 9 10 11 12 15 16; do echo "T=$T"; GQ_DSTEP=1 CUDA_LAUNCH_BLOCKING=1 timeout 120 python tools/_shapes.py one 3 3 $T 2>&1 | tail -1; done
