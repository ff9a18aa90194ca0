# usage: bash scripts/gpu_check.sh [tag]  -- smoke, GPU tests, bench (runs on the B200 box)
set -x
R=${1:-dev}
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv
python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke_$R.log 2>&1; echo smoke rc=$?
timeout 1200 python -m pytest tests -m gpu -q --maxfail=30 -p no:cacheprovider > gpurun_out/pytest_gpu_$R.log 2>&1; echo pytest rc=$?
timeout 900 python bench.py --steps 10 --warmup 3 --cpu-seconds 10 > gpurun_out/bench_$R.json 2> gpurun_out/bench_$R.err; echo bench rc=$?
tail -5 gpurun_out/pytest_gpu_$R.log
cat gpurun_out/bench_$R.json
