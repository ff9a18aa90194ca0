set -x
rm -f gpurun_out/bs6_run.log
SB200_BS6_RUN=16 timeout 600 python -m pytest tests/test_gpu_gs.py -q -x -p no:cacheprovider 2>&1 | tail -2 >> gpurun_out/bs6_run.log
SB200_BS6_RUN=0 timeout 600 python -m pytest tests/test_gpu_gs.py -q -x -p no:cacheprovider 2>&1 | tail -2 >> gpurun_out/bs6_run.log
for r in 1 2 4 16 64 0; do echo "run=$r" >> gpurun_out/bs6_run.log; SB200_BS6_RUN=$r timeout 300 python scripts/expt/time_bs6.py 2 3 5 7 15 >> gpurun_out/bs6_run.log 2>&1; done
cat gpurun_out/bs6_run.log
