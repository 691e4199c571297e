# Round-2 evidence in one GPU session (each step only after the previous one
# exited; numbers printed under a profiler are never bench values):
#   sanitizers over every kernel family, the default bench line, the reference
#   arm, the secondary lines, the ncu launch list of the default bench and one
#   `ncu --set full` capture of the headline kernel (C5 mul_add).
set -u
mkdir -p gpurun_out/ev
S=gpurun_out/ev
if [ "${SAN:-1}" = 1 ]; then
  for tool in memcheck racecheck synccheck initcheck; do
    timeout 1200 compute-sanitizer --tool $tool --error-exitcode 9 python tools/sanitize_kernels.py > $S/san_$tool.log 2>&1
    echo "sanitizer $tool rc=$?"; tail -2 $S/san_$tool.log
  done
  for tool in memcheck racecheck; do
    BFP_BULK=2 timeout 1200 compute-sanitizer --tool $tool --error-exitcode 9 python tools/sanitize_kernels.py --bulk > $S/san_bulk_$tool.log 2>&1
    echo "sanitizer bulk $tool rc=$?"; tail -2 $S/san_bulk_$tool.log
  done
fi
if [ "${BENCH:-1}" = 1 ]; then
  timeout 900 python bench.py > $S/bench_default.jsonl 2> $S/bench_default.err; echo "bench default rc=$?"
  timeout 900 python bench.py --impl reference > $S/bench_reference.jsonl 2> $S/bench_reference.err; echo "bench reference rc=$?"
  timeout 1200 python bench.py --config X1,X2,X3,X3u --no-cpu-baseline > $S/bench_secondary.jsonl 2> $S/bench_secondary.err; echo "bench secondary rc=$?"
fi
if [ "${NCU:-1}" = 1 ]; then
  timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file $S/launches_default.csv \
    python bench.py --steps 2 --warmup 3 --no-e2e --no-cpu-baseline --no-ncu > $S/launches_default.log 2>&1; echo "launch list rc=$?"
  # the report goes to /tmp first: gpurun_out/ is size-capped, so the raw page is exported here and the
  # .ncu-rep only copied when it is small enough
  timeout 900 ncu --set full --clock-control none --import-source on -k regex:k_arith -c 1 -o /tmp/c5_full -f \
    python tools/profile_kernels.py --config C5 --iters 1 > $S/c5_full.log 2>&1; echo "ncu full C5 rc=$?"
  ncu -i /tmp/c5_full.ncu-rep --page raw --csv > $S/c5_full_raw.csv 2>/dev/null
  [ "$(stat -c %s /tmp/c5_full.ncu-rep 2>/dev/null || echo 99999999)" -lt 40000000 ] && cp /tmp/c5_full.ncu-rep $S/c5_full.ncu-rep
  timeout 900 ncu --set full --clock-control none --import-source on -k regex:k_arith --launch-skip 9 -c 1 -o $S/c4_mul815_full -f \
    python tools/profile_kernels.py --config C4 --iters 1 > $S/c4_full.log 2>&1; echo "ncu full C4 1/8/15 mul rc=$?"
fi
