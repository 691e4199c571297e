# One GPU session: bench (all configs, default mode + RZ/FTZ secondary rows),
# launch list of the default bench, ncu --set full of chosen dominant kernels.
# ncu reports stay in /tmp on the box (too large to bring back); their raw-page
# summaries and details pages go to gpurun_out/ncu/.
#   PROF="c1_add:C1:add ..." bash tools/gpu_prof.sh
set -u
mkdir -p gpurun_out/ncu /tmp/ncu
if [ "${BENCH:-1}" = 1 ]; then
timeout 300 python bench.py --config C1,C2 --no-e2e --no-cpu-baseline > gpurun_out/bench_quick.jsonl 2> gpurun_out/bench_quick.err; echo quick_rc=$?; tail -3 gpurun_out/bench_quick.err
timeout 900 python bench.py --config all --steps 50 --warmup 5 > gpurun_out/bench_all.jsonl 2> gpurun_out/bench_all.err; echo bench_all_rc=$?
timeout 300 python bench.py --config C1,C2,C4 --rounding rz --no-e2e --no-cpu-baseline > gpurun_out/bench_rz.jsonl 2> gpurun_out/bench_rz.err; echo bench_rz_rc=$?
timeout 300 python bench.py --config C1,C2,C4 --subnormals ftz --no-e2e --no-cpu-baseline > gpurun_out/bench_ftz.jsonl 2> gpurun_out/bench_ftz.err; echo bench_ftz_rc=$?
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/ncu/launches_default.csv python bench.py --steps 2 --warmup 3 --no-e2e --no-cpu-baseline > gpurun_out/ncu/launches_default.log 2>&1; echo launches_rc=$?
fi
for spec in ${PROF:-}; do
  IFS=: read name cfg ops <<< "$spec"
  timeout 600 ncu --set full --clock-control none --import-source on -k regex:k_arith -s 1 -c 1 \
    -o /tmp/ncu/$name -f python tools/profile_kernels.py --config $cfg --ops $ops --iters 3 > gpurun_out/ncu/$name.log 2>&1; echo prof_${name}_rc=$?
  ncu -i /tmp/ncu/$name.ncu-rep --page details > gpurun_out/ncu/$name.details.txt 2>&1
done
if [ -n "${PROF:-}" ]; then
python tools/ncu_summary.py gpurun_out/ncu/summary.json /tmp/ncu/*.ncu-rep > gpurun_out/ncu/summary.txt 2>&1; echo summary_rc=$?
fi
for f in gpurun_out/*.jsonl; do echo "== $f"; python3 -c "
import json,sys
for l in open('$f'):
    d=json.loads(l); r=d['roofline']; print(d['config']['workload'][:3], d['value'], 'step_frac', r['step']['frac'], 'eager_ms', r['step'].get('ms_per_step_eager'), d['clocks']['sm_mhz'], 'e2e', d.get('e2e',{}).get('value'), 'cpu', d.get('cpu_baseline',{}).get('value'))
    for k,v in r['per_op'].items(): print('   ',k, v['ms'], v['gelem_s'], v['hbm_frac'], v.get('logic_frac'), v.get('logic_frac_sustained'), v.get('binding'), v.get('frac_of_binding'))
"; done
