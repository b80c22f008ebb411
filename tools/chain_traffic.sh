# DRAM bytes + duration of the chain sweeps of one step for several residency caps
mkdir -p gpurun_out/ct
for w in 6 8 12 0; do
  GQ_CHAIN_WARPS=$w ncu --metrics dram__bytes_read.sum,dram__bytes_write.sum,gpu__time_duration.sum --clock-control none -k regex:k_chain --launch-skip 4 -c 4 --csv --log-file gpurun_out/ct/w$w.csv python tools/stepprof.py > /dev/null 2>&1
done
