# round-2 profile: NVTX-scoped launch list of the bench step, ncu --set full
# of the seven bench kernels and of the BS6 product kernel at config 3's N=1/2
set -x
R=r02
ncu --nvtx --nvtx-include "timed/" --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none --csv --log-file gpurun_out/launches_$R.csv python bench.py --steps 2 --warmup 3 --no-e2e --no-cpu-baseline --no-extras > gpurun_out/launches_bench_$R.log 2>&1; echo launches rc=$?
ncu --set full --import-source on --clock-control none -k regex:'k_elem|k_lattice|k_bs6|k_bs7' -s 7 -c 7 -o gpurun_out/prof_$R -f python scripts/profile_kernels.py > gpurun_out/prof_$R.log 2>&1; echo full rc=$?
for p in 1 2; do ncu --set full --import-source on --clock-control none -k regex:k_bs6 -s 2 -c 1 -o gpurun_out/prof_${R}_bs6_N$p -f python scripts/profile_bs6_low.py $p > gpurun_out/prof_${R}_bs6_N$p.log 2>&1; echo bs6 N=$p rc=$?; done
