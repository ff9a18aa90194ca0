set -x
rm -f gpurun_out/bs6_ab11.log
SB200_BS6_CFG=map,10 timeout 600 python -m pytest tests/test_gpu_gs.py -q -x -p no:cacheprovider 2>&1 | tail -2 >> gpurun_out/bs6_ab11.log
for c in default map,8 map,10 map,12; do SB200_BS6_CFG=$c timeout 300 python scripts/expt/time_bs6.py 1 2 3 4 5 7 10 15 >> gpurun_out/bs6_ab11.log 2>&1; done
cat gpurun_out/bs6_ab11.log
