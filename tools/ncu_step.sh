# ncu --set full of one whole PCGM step at the headline (the second step of tools/stepprof.py:
# the regex skips pcg_start's initial preconditioner -- 4 sweeps + 1 outer rhs -- and the 7
# kernels of step 1)
OUT=${1:-step}
export STEPS=3
python tools/stepprof.py > gpurun_out/sp.log 2>&1 && \
ncu --set full --clock-control none --import-source on -k regex:"^(k_dstep|k_rstep|k_update_x|k_chain|k_chainm|k_grid|k_dirupdate|k_dirupdate_x)$" \
    --launch-skip 12 -c 7 -o gpurun_out/$OUT python tools/stepprof.py > gpurun_out/ncu_$OUT.log 2>&1
tail -3 gpurun_out/ncu_$OUT.log
