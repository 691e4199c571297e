set -x
timeout 1200 python -m pytest tests -x -q -m gpu > gpurun_out/pytest_gpu.log 2>&1; echo pytest_rc=$?
tail -5 gpurun_out/pytest_gpu.log
timeout 1500 python bench.py --config all --steps 20 --warmup 3 > gpurun_out/bench_all.log 2> gpurun_out/bench_all.err; echo bench_rc=$?
tail -5 gpurun_out/bench_all.err
