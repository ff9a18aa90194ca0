timeout 400 python -m pytest tests/test_gpu_bs6_sweep.py -x -q -p no:cacheprovider -k "not c3" > gpurun_out/sweep_t.log 2>&1; echo rc=$?; tail -1 gpurun_out/sweep_t.log
CFGS="${CFGS:-0,-1,0,-1;3,0,0,-1}" timeout 300 python scripts/expt/time_bs6_sweep.py 1 2 2>&1 | tee gpurun_out/sweep_time.log
CFGS="0,-1,0,-1" timeout 300 ncu --set full --clock-control none --import-source on -k regex:k_bs6_sweep -s 2 -c 1 -o gpurun_out/sweep_p1x -f python scripts/expt/time_bs6_sweep.py 1 > gpurun_out/ncu_sweep.log 2>&1; echo ncu=$?
