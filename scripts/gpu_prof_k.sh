# usage: bash scripts/gpu_prof_k.sh <tag> <kernel-regex> <count> [profile_kernels args]
set -x
R=$1; K=$2; C=${3:-2}; shift 3
ncu --set full --import-source on --clock-control none -k regex:"$K" -c $C -o gpurun_out/prof_$R python scripts/profile_kernels.py "$@" > gpurun_out/prof_$R.log 2>&1; echo full rc=$?
tail -3 gpurun_out/prof_$R.log
