# A/B: BS6 default (lanes/pairs) vs TMA-fed lanes kernel (10: no swizzle, 11: swizzle)
set -x
rm -f gpurun_out/bs6_ab6.log
for k in 10 11; do SB200_BS6_KERNEL=$k timeout 600 python -m pytest tests/test_gpu_gs.py tests/test_gpu_dist.py -q -x -p no:cacheprovider 2>&1 | tail -2 >> gpurun_out/bs6_ab6.log; done
for k in 0 10 11; do SB200_BS6_KERNEL=$k timeout 300 python scripts/expt/time_bs6.py 1 2 3 5 7 10 15 >> gpurun_out/bs6_ab6.log 2>&1; done
SB200_BS6_KERNEL=11 timeout 300 ncu --set full --import-source on --clock-control none -k regex:k_bs6 -s 2 -c 1 -o gpurun_out/bs6_v11_n7 python scripts/expt/time_bs6.py 7 > /dev/null 2>&1
cat gpurun_out/bs6_ab6.log
