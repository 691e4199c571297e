for v in early late; do
cp tools/variants/lib_$v.so paper_1602_04716_b200/libbfpgpu.so
for p in 1 0; do
BFP_PDL=$p timeout 900 python bench.py --config C2,C4,C5,C3 --steps 30 --warmup 5 --no-cpu-baseline --no-e2e > gpurun_out/b.log 2>/dev/null
python3 -c "
import json
for l in open('gpurun_out/b.log'):
    d=json.loads(l); r=d['roofline']; print('$v PDL=$p', d['config']['workload'][:3], d['value'], d['ms_per_step'], r['step']['ms_per_step_with_kernel_events'], d['clocks']['sm_mhz'])
"
done; done
