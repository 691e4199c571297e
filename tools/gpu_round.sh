set -x
timeout 1500 python -m pytest tests -q -x -m gpu > gpurun_out/pytest_gpu.log 2>&1; echo pytest_rc=$?
tail -3 gpurun_out/pytest_gpu.log
timeout 900 python bench.py --config C3 --steps 20 --warmup 3 --no-cpu-baseline --no-e2e > gpurun_out/bench_c3.log 2> gpurun_out/bench_c3.err; echo bench_rc=$?
