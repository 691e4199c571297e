BFP_PDL=1 timeout 900 python bench.py --config C3 --steps 20 --warmup 5 --no-cpu-baseline --no-e2e > gpurun_out/bench_c3p.log 2> gpurun_out/bench_c3p.err; echo rc=$?
tail -30 gpurun_out/bench_c3p.err
