timeout 1500 python -m pytest tests -q -x -m "gpu" > gpurun_out/pytest_gpu.log 2>&1; echo pytest_rc=$?
tail -2 gpurun_out/pytest_gpu.log
