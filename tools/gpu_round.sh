timeout 1800 python -m pytest tests -q -x -m "gpu" > gpurun_out/pytest_gpu.log 2>&1; echo pytest_rc=$?
tail -2 gpurun_out/pytest_gpu.log
timeout 1500 python bench.py --config C3,C5 --steps 30 --warmup 5 --no-cpu-baseline --no-e2e > gpurun_out/b.log 2>/dev/null; echo bench_rc=$?
python3 -c "
import json
for l in open('gpurun_out/b.log'):
    d=json.loads(l); r=d['roofline']; print(d['config']['workload'][:3], d['value'], 'step_frac', r['step']['frac'], d['clocks']['sm_mhz'])
    for k,v in r['per_op'].items(): print('   ',k, v['ms'], v['gelem_s'], v['hbm_frac'], v.get('logic_frac'), v.get('binding'), v.get('frac_of_binding'))
"
