# A/B: BS6 kernel variants 3 (lean), 5 (lean2: int4 ids), 6 (lean2 + swizzle always)
set -x
rm -f gpurun_out/bs6_ab5.log
for k in 7 9; do SB200_BS6_KERNEL=$k timeout 600 python -m pytest tests/test_gpu_gs.py tests/test_gpu_dist.py -q -x -p no:cacheprovider 2>&1 | tail -2 >> gpurun_out/bs6_ab5.log; done
for k in 3 7 8 9; do SB200_BS6_KERNEL=$k timeout 300 python scripts/expt/time_bs6.py 1 2 3 5 7 10 15 >> gpurun_out/bs6_ab5.log 2>&1; done
SB200_BS6_KERNEL=7 timeout 300 ncu --set full --import-source on --clock-control none -k regex:k_bs6 -s 2 -c 1 -o gpurun_out/bs6_v7_n7 python scripts/expt/time_bs6.py 7 > /dev/null 2>&1
cat gpurun_out/bs6_ab5.log
