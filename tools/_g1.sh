set -x
python -m pytest tests/test_gpu_parity.py tests/test_gpu_variants.py tests/test_gpu_boundary.py -x -q > gpurun_out/t_orhs.log 2>&1; tail -3 gpurun_out/t_orhs.log
for v in "" "GQ_NO_ORHS=1" "GQ_FUSE_X=1" ""; do
  env $v python bench.py --steps 100 --warmup 5 --no-cpu-baseline > gpurun_out/b_orhs_${v%%=*}.json 2>gpurun_out/b_orhs.err; tail -c 600 gpurun_out/b_orhs_${v%%=*}.json | head -c 300; echo
done
python -m pytest tests/test_gpu_fullsize.py -x -q -k headline > gpurun_out/t_fs.log 2>&1; tail -2 gpurun_out/t_fs.log
