timeout 1500 python -m pytest tests -q -x -m "gpu" > gpurun_out/pytest_gpu.log 2>&1; echo pytest_rc=$?
tail -2 gpurun_out/pytest_gpu.log
for p in 1 0 1 0; do
BFP_PDL=$p timeout 900 python bench.py --config C3,C1,C2 --steps 30 --warmup 5 --no-cpu-baseline --no-e2e > gpurun_out/bench_p$p.log 2>/dev/null
python3 -c "
import json,sys
for l in open('gpurun_out/bench_p$p.log'):
    d=json.loads(l); print('PDL=$p', d['config']['workload'][:3], d['value'], d['ms_per_step'], d['clocks']['sm_mhz'], {k:(v['ms'],v['hbm_frac']) for k,v in d['roofline']['per_op'].items()})
"
done
