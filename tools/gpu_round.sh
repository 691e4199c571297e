timeout 1800 python -m pytest tests -q -x -m "gpu" > gpurun_out/pytest_gpu.log 2>&1; echo pytest_rc=$?
tail -3 gpurun_out/pytest_gpu.log
