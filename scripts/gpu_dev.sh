set -x
timeout 600 python -m pytest tests/test_gpu_cg_device.py -q -x -p no:cacheprovider > gpurun_out/cgdev.log 2>&1; echo cg rc=$?
timeout 900 python -m pytest tests -m gpu -q -p no:cacheprovider > gpurun_out/pytest_all.log 2>&1; echo all rc=$?
timeout 300 python scripts/expt/run_bs5.py > gpurun_out/bs5.log 2>&1
SB200_NO_TMA=1 timeout 300 python scripts/expt/run_bs5.py >> gpurun_out/bs5.log 2>&1
tail -30 gpurun_out/cgdev.log; tail -3 gpurun_out/pytest_all.log; cat gpurun_out/bs5.log
