set -x
rm -f gpurun_out/bs6_single.log
SB200_BS6_CFG=single,0,10 timeout 600 python -m pytest tests/test_gpu_gs.py tests/test_gpu_dist.py -q -x -p no:cacheprovider 2>&1 | tail -2 >> gpurun_out/bs6_single.log
timeout 300 python scripts/expt/time_bs6.py 3 5 7 10 15 >> gpurun_out/bs6_single.log 2>&1
for c in single,0,10 single,1,10 single,0,12 single,0,8 single,1,8; do SB200_BS6_CFG=$c timeout 300 python scripts/expt/time_bs6.py 3 5 7 10 15 >> gpurun_out/bs6_single.log 2>&1; done
cat gpurun_out/bs6_single.log
