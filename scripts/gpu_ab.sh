# A/B: BS7 int4 kernel (0) vs lanes (1: 128x8, 2: 256x4) vs pairs (3: 128x4, 4: 128x8)
set -x
rm -f gpurun_out/bs7_ab3.log
for k in 9; do SB200_BS7_KERNEL=$k timeout 600 python -m pytest tests/test_gpu_gs.py -q -x -p no:cacheprovider 2>&1 | tail -2 >> gpurun_out/bs7_ab3.log; done
for k in 9 5 6 7 8; do SB200_BS7_KERNEL=$k timeout 300 python scripts/expt/time_bs7.py 1 2 3 4 5 6 7 10 15 >> gpurun_out/bs7_ab3.log 2>&1; done
cat gpurun_out/bs7_ab3.log
