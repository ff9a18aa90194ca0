set -x
timeout 600 python -m pytest tests/test_gpu_gs.py tests/test_gpu_dist.py tests/test_gpu_cg_device.py -q -x -p no:cacheprovider 2>&1 | tail -2 > gpurun_out/bs6_final.log
timeout 300 python scripts/expt/time_bs6.py 1 2 3 4 5 6 7 8 10 12 15 >> gpurun_out/bs6_final.log 2>&1
cat gpurun_out/bs6_final.log
