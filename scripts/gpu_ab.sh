# A/B: BS6 default vs one-super-block-per-CTA (20/21: 12 CTA/SM bound, 22/23: 16; odd = swizzle)
set -x
rm -f gpurun_out/bs6_ab7.log
for k in 21; do SB200_BS6_KERNEL=$k timeout 600 python -m pytest tests/test_gpu_gs.py -q -x -p no:cacheprovider 2>&1 | tail -2 >> gpurun_out/bs6_ab7.log; done
for k in 0 20 21 22 23; do SB200_BS6_KERNEL=$k timeout 300 python scripts/expt/time_bs6.py 1 2 3 5 7 10 15 >> gpurun_out/bs6_ab7.log 2>&1; done
cat gpurun_out/bs6_ab7.log
