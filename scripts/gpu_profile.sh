# usage: bash scripts/gpu_profile.sh [tag] -- launch list (NVTX-scoped bench) + ncu --set full of the 7 kernels + sweeps
set -x
R=${1:-r01}
ncu --nvtx --nvtx-include "timed/" --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none --csv --log-file gpurun_out/launches_$R.csv python bench.py --steps 2 --warmup 3 --no-e2e --no-cpu-baseline > gpurun_out/launches_bench_$R.log 2>&1; echo launches rc=$?
ncu --set full --import-source on --clock-control none -k regex:'k_elem|k_lattice|k_bs6|k_bs7' -s 7 -c 7 -o gpurun_out/prof_$R python scripts/profile_kernels.py > gpurun_out/prof_$R.log 2>&1; echo full rc=$?
timeout 1500 python scripts/sweep.py --out gpurun_out/sweep_$R --points 40 --trials 10 > gpurun_out/sweep_$R.log 2>&1; echo sweep rc=$?
tail -30 gpurun_out/sweep_$R.log
