nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv
timeout 1800 python -m pytest tests -q -x -m "gpu" --durations=15 > gpurun_out/pytest_gpu.log 2>&1; echo pytest_rc=$?
tail -25 gpurun_out/pytest_gpu.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke.log 2>&1; echo smoke_rc=$?; tail -2 gpurun_out/smoke.log
timeout 600 python bench.py > gpurun_out/bench_default.log 2>gpurun_out/bench_default.err; echo bench_rc=$?
cat gpurun_out/bench_default.log | cut -c1-400
timeout 1500 python bench.py --config all --steps 30 --warmup 5 > gpurun_out/bench_all.log 2>gpurun_out/bench_all.err; echo benchall_rc=$?
