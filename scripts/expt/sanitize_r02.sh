#!/bin/bash
# compute-sanitizer over the round-2 BS6 kernels (scripts/expt/sanitize_r02.py)
CS=/usr/local/cuda/bin/compute-sanitizer
python scripts/expt/sanitize_r02.py > gpurun_out/san_plain.log 2>&1; echo plain rc=$?
for tool in memcheck synccheck; do
  timeout 900 $CS --tool $tool --print-limit 50 python scripts/expt/sanitize_r02.py > gpurun_out/san_$tool.log 2>&1; echo $tool rc=$?
done
for part in tiled sweep halo; do
  timeout 900 $CS --tool racecheck --racecheck-report hazard --print-limit 20 python scripts/expt/sanitize_r02.py $part > gpurun_out/san_racecheck_$part.log 2>&1; echo racecheck $part rc=$?
done
timeout 900 $CS --tool memcheck python -m pytest tests/test_gpu_bs6_tiled.py tests/test_gpu_halo.py -x -q > gpurun_out/san_memcheck_tests.log 2>&1; echo memcheck tests rc=$?
