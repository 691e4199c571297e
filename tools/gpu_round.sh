timeout 1500 python -m pytest tests -q -x -m "gpu" > gpurun_out/pytest_gpu.log 2>&1; echo pytest_rc=$?
tail -2 gpurun_out/pytest_gpu.log
timeout 900 python bench.py --config C2,C3,C4,C5,C1 --steps 30 --warmup 5 --no-cpu-baseline --no-e2e > gpurun_out/bench_gen.log 2>/dev/null; echo bench_rc=$?
python3 -c "
import json,sys
for l in open('gpurun_out/bench_gen.log'):
    d=json.loads(l); print(d['config']['workload'][:3], d['value'], d['ms_per_step'], d['clocks']['sm_mhz'], d['clocks']['reasons'])
    for k,v in d['roofline']['per_op'].items(): print('   ',k, v['ms'], v['gelem_s'], v['hbm_frac'], v.get('logic_frac'), v.get('binding'), v.get('frac_of_binding'))
"
