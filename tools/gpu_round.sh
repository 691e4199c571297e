for r in 1 2; do
for ev in 1 0; do
for p in 1 0; do
BFP_PDL=$p BFP_BENCH_KERNEL_EVENTS=$ev timeout 900 python bench.py --config C2,C1 --steps 100 --warmup 5 --no-cpu-baseline --no-e2e > gpurun_out/b.log 2>/dev/null
python3 -c "
import json
for l in open('gpurun_out/b.log'):
    d=json.loads(l); print('EV=$ev PDL=$p', d['config']['workload'][:3], d['value'], d['ms_per_step'], d['clocks']['sm_mhz'])
"
done; done; done
