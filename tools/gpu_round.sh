timeout 1800 python -m pytest tests -q -x -m "gpu" > gpurun_out/pytest_gpu.log 2>&1; echo pytest_rc=$?
tail -2 gpurun_out/pytest_gpu.log
timeout 1500 python bench.py --config all --steps 50 --warmup 5 > gpurun_out/bench_all.log 2> gpurun_out/bench_all.err; echo bench_rc=$?
python3 -c "
import json
for l in open('gpurun_out/bench_all.log'):
    d=json.loads(l); r=d['roofline']; print(d['config']['workload'][:3], d['value'], 'step_frac', r['step']['frac'], 'kern frac', r['frac'], 'e2e', d.get('e2e',{}).get('value'), d.get('e2e',{}).get('frac_of_pcie_bound'), 'cpu', d.get('cpu_baseline',{}).get('value'), d['clocks']['sm_mhz'], d['clocks']['reasons'])
"
timeout 900 python bench.py --impl reference > gpurun_out/bench_ref.log 2>&1; echo ref_rc=$?
python3 -c "
import json
for l in open('gpurun_out/bench_ref.log'):
    d=json.loads(l); print('REF', d['value'], d['cpu_baseline']['cores'], d['cpu_baseline']['per_op'])
"
