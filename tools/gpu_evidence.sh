# Round evidence in one GPU session: parity suite, smoke, default bench, all
# configs, launch list of the default bench, and one `ncu --set full` capture
# per config holding every timed kernel (traffic -> profiles/ncu_traffic.json
# via tools/ncu_traffic.py; reports stay in /tmp on the box, raw summaries come back).
set -u
mkdir -p gpurun_out/ncu /tmp/ncu
if [ "${TESTS:-1}" = 1 ]; then
timeout 1500 python -m pytest tests -q -x -m gpu > gpurun_out/pytest_gpu.log 2>&1; echo pytest_rc=$?; tail -2 gpurun_out/pytest_gpu.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke.log 2>&1; echo smoke_rc=$?; tail -1 gpurun_out/smoke.log
fi
if [ "${BENCH:-1}" = 1 ]; then
timeout 600 python bench.py --impl reference > gpurun_out/bench_reference.jsonl 2> gpurun_out/bench_reference.err; echo bench_reference_rc=$?
timeout 600 python bench.py > gpurun_out/bench_default.jsonl 2> gpurun_out/bench_default.err; echo bench_default_rc=$?
timeout 900 python bench.py --config all --steps 50 --warmup 5 > gpurun_out/bench_all.jsonl 2> gpurun_out/bench_all.err; echo bench_all_rc=$?
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/ncu/launches_default.csv python bench.py --steps 2 --warmup 3 --no-e2e --no-cpu-baseline > gpurun_out/ncu/launches_default.log 2>&1; echo launches_rc=$?
fi
ARGS=""
for cfg in ${CFGS:-C1 C2 C3 C4 C5}; do
  case $cfg in C3) K='regex:k_(arith|pack_f32|unpack_f32)';; X3) K='regex:bfp_chain_k';; *) K='regex:k_arith';; esac
  timeout 900 ncu --set full --clock-control none --import-source on -k "$K" \
    -o /tmp/ncu/$cfg -f python tools/profile_kernels.py --config $cfg --iters 1 > gpurun_out/ncu/$cfg.log 2>&1; echo prof_${cfg}_rc=$?
  ARGS="$ARGS $cfg=/tmp/ncu/$cfg.ncu-rep"
done
cp profiles/ncu_traffic.json gpurun_out/ncu/ncu_traffic.json 2>/dev/null
python tools/ncu_traffic.py gpurun_out/ncu/ncu_traffic.json $ARGS > gpurun_out/ncu/traffic.txt 2>&1; echo traffic_rc=$?; cat gpurun_out/ncu/traffic.txt
python tools/ncu_summary.py gpurun_out/ncu/summary.json /tmp/ncu/*.ncu-rep > gpurun_out/ncu/summary.txt 2>&1; echo summary_rc=$?
