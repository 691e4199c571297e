set -x
timeout 300 python bench.py --steps 50 --warmup 5 > gpurun_out/bench.log 2> gpurun_out/bench.err; echo bench_rc=$?
tail -3 gpurun_out/bench.log; tail -30 gpurun_out/bench.err
