set -x
rm -f gpurun_out/bs6_deep.log
SB200_BS6_CFG=deep,0,8 timeout 600 python -m pytest tests/test_gpu_gs.py -q -x -p no:cacheprovider 2>&1 | tail -2 >> gpurun_out/bs6_deep.log
timeout 300 python scripts/expt/time_bs6.py 2 3 5 7 15 >> gpurun_out/bs6_deep.log 2>&1
for c in deep,0,8 deep,0,10 deep,0,6 deep,1,8; do SB200_BS6_CFG=$c timeout 300 python scripts/expt/time_bs6.py 2 3 5 7 15 >> gpurun_out/bs6_deep.log 2>&1; done
cat gpurun_out/bs6_deep.log
