set -x
timeout 300 python scripts/expt/run_bs6_diag.py > gpurun_out/diag_bs6.log 2>&1; echo diag rc=$?
timeout 900 python scripts/sweep.py --out gpurun_out/sweep_vec_r01 --tests bs1,bs2,bs3,bs4,bs5 --points 40 --trials 10 > gpurun_out/sweep_vec.log 2>&1; echo sweep rc=$?
timeout 600 ncu --set full --import-source on --clock-control none -k regex:'k_lattice|k_bs6' -s 5 -c 3 -o gpurun_out/prof_r01c python scripts/profile_kernels.py > gpurun_out/prof_r01c.log 2>&1; echo full rc=$?
cat gpurun_out/diag_bs6.log; tail -12 gpurun_out/sweep_vec.log
