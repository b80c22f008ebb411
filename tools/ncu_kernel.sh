# ncu --set full of one kernel family of the PCGM step at the headline (tools/stepprof.py)
# usage: bash tools/ncu_kernel.sh <regex> <out-name> [count]
K=$1; OUT=$2; C=${3:-2}
export STEPS=3
python tools/stepprof.py > gpurun_out/sp_$OUT.log 2>&1 && \
ncu --set full --clock-control none --import-source on -k regex:$K --launch-skip 2 -c $C -o gpurun_out/$OUT python tools/stepprof.py > gpurun_out/ncu_$OUT.log 2>&1
tail -3 gpurun_out/ncu_$OUT.log
