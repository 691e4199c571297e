# A/B of the bulk-copy ring depth on the GPU box (rebuilds in the box's scratch copy).
set -u
mkdir -p gpurun_out
run() {  # tag
  timeout 400 python bench.py --config C3,C4,C5 --steps 30 --no-e2e --no-cpu-baseline > gpurun_out/ab_$1.jsonl 2> gpurun_out/ab_$1.err; echo "ab_$1 rc=$?"
  python3 -c "
import json
for l in open('gpurun_out/ab_$1.jsonl'):
    d=json.loads(l)
    for k,v in d['roofline']['per_op'].items():
        if 'mul' in k: print('$1', k, v['ms'], v['gelem_s'], v['hbm_frac'], v.get('logic_frac'), v.get('frac_of_binding'))
"
}
run base
BFP_BULK=0 run plain
for b in 8192 12288; do
  BFP_EXTRA_NVCC="-DBFP_BULK_BUDGET=$b" python -c "from paper_1602_04716_b200.build import build; build(force=True)" > gpurun_out/build_$b.log 2>&1; echo build_$b rc=$?
  run b$b
done
