#!/bin/bash
# p=2 z-sweep row-lane consumer: parity tests + A/B timing (one gpurun call)
set -x
mkdir -p gpurun_out
timeout 600 python -m pytest tests/test_gpu_bs6_sweep.py -x -q 2>&1 | tail -5
CFGS="${CFGS:-0,-1,0,-1;3,-1,0,-1;3,-1,0,-1,7;6,-1,0,-1,16}" timeout 300 python scripts/expt/time_bs6_sweep.py 2
if [ -n "$NCU" ]; then
SB200_BS6_SWEEP=1 timeout 600 ncu --set full --import-source on --clock-control none -k regex:k_bs6_sweep2 -s 1 -c 1 -o gpurun_out/sweep2 -f python scripts/profile_bs6_low.py 2
fi
