timeout 1500 python -m pytest tests -q -m "gpu" > gpurun_out/pytest_gpu.log 2>&1; echo pytest_rc=$?
tail -2 gpurun_out/pytest_gpu.log
timeout 1500 python bench.py --config all --steps 30 --warmup 5 > gpurun_out/bench_all.log 2> gpurun_out/bench_all.err; echo bench_rc=$?
python3 -c "
import json
for l in open('gpurun_out/bench_all.log'):
    d=json.loads(l); print(d['config']['workload'][:3], d['value'], d['roofline']['frac'], d.get('e2e',{}).get('value'), d.get('e2e',{}).get('frac_of_pcie_bound'), d.get('cpu_baseline',{}).get('value'), d['clocks'])
    for k,v in d['roofline']['per_op'].items(): print('   ',k, v['ms'], v['gelem_s'], v['hbm_frac'], v.get('logic_frac'), v.get('binding'), v.get('frac_of_binding'))
"
timeout 600 python bench.py --steps 3 --warmup 3 --no-cpu-baseline --no-e2e > gpurun_out/plain_bench.log 2>&1 && ncu --metrics gpu__time_duration.sum --clock-control none -k regex:k_ --csv --log-file gpurun_out/launches_bench_default.csv python bench.py --steps 3 --warmup 3 --no-cpu-baseline --no-e2e > /dev/null 2>&1; echo ncu_rc=$?
