mkdir -p gpurun_out/ct
for v in 1 0; do
  GQ_DD=$v ncu --metrics dram__bytes_read.sum,dram__bytes_write.sum,gpu__time_duration.sum,sm__warps_active.avg.pct_of_peak_sustained_active,l1tex__data_pipe_lsu_wavefronts.avg.pct_of_peak_sustained_elapsed --clock-control none -k regex:k_chain --launch-skip 4 -c 4 --csv --log-file gpurun_out/ct/dd$v.csv python tools/stepprof.py > /dev/null 2>&1
done
