set -x
timeout 1500 python -m pytest tests -q -m gpu > gpurun_out/pytest_gpu.log 2>&1; echo pytest_rc=$?
tail -5 gpurun_out/pytest_gpu.log
timeout 900 python bench.py --config C3,C1,C2 --steps 20 --warmup 3 --no-cpu-baseline > gpurun_out/bench_c3.log 2> gpurun_out/bench_c3.err; echo bench_rc=$?
tail -3 gpurun_out/bench_c3.err
