set -x
rm -f gpurun_out/bs6_ab12.log
for c in lanes,0,12 lanes,1,12 lanes,0,10 lanes,1,10 lanes,0,8 lanes,1,8 lanes,1,6 lanes,0,6; do SB200_BS6_CFG=$c timeout 300 python scripts/expt/time_bs6.py 3 4 >> gpurun_out/bs6_ab12.log 2>&1; done
cat gpurun_out/bs6_ab12.log
