# Round-end evidence in one GPU session: GPU parity suite, smoke, default bench,
# all configs (+ RZ / FTZ rows), launch list, ncu --set full of each config's
# dominant kernel (summaries only; reports stay in /tmp on the box).
set -u
mkdir -p gpurun_out/ncu
timeout 900 python -m pytest tests -q -x -m gpu > gpurun_out/pytest_gpu.log 2>&1; echo pytest_rc=$?; tail -2 gpurun_out/pytest_gpu.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke.log 2>&1; echo smoke_rc=$?; tail -1 gpurun_out/smoke.log
timeout 600 python bench.py > gpurun_out/bench_default.jsonl 2> gpurun_out/bench_default.err; echo bench_default_rc=$?
PROF="c1_add:C1:add c2_mul:C2:mul c3_mul:C3:mul c4_mul_8_15:C4:mul_1/8/15 c4_mul_5_7:C4:mul_1/5/7 c5_mul_add:C5:mul_add" bash tools/gpu_prof.sh
