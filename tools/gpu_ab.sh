# A/B of build / runtime variants on the GPU box (rebuilds in the box's scratch
# copy; the repo's own .so is restored at the end).
#   VARIANTS="base:: minb6::-DBFP_ARITH_MINB=6 bulk:BFP_BULK=1:" CONFIGS=C3,C4,C5 bash tools/gpu_ab.sh
# each variant = tag:ENV_ASSIGNMENTS(comma-separated):NVCC_FLAGS
set -u
mkdir -p gpurun_out
cp paper_1602_04716_b200/libbfpgpu.so /tmp/libbfpgpu.orig.so
for v in $VARIANTS; do
  IFS=: read tag envs flags <<< "$v"
  if [ -n "$flags" ]; then
    BFP_EXTRA_NVCC="$flags" python -c "from paper_1602_04716_b200.build import build; build(force=True)" > gpurun_out/build_$tag.log 2>&1; echo build_$tag rc=$?
  else
    cp /tmp/libbfpgpu.orig.so paper_1602_04716_b200/libbfpgpu.so
  fi
  env $(echo $envs | tr ',' ' ') timeout 600 python bench.py --config ${CONFIGS:-C3,C4,C5} --steps 30 --no-e2e --no-cpu-baseline > gpurun_out/ab_$tag.jsonl 2> gpurun_out/ab_$tag.err; echo "ab_$tag rc=$?"
  python3 -c "
import json
for l in open('gpurun_out/ab_$tag.jsonl'):
    d=json.loads(l)
    for k,v in d['roofline']['per_op'].items():
        print('$tag', k, v['ms'], v['gelem_s'], v['hbm_frac'], v.get('logic_frac'), v.get('logic_frac_at_load_clock'), v.get('frac_of_binding'))
"
done
cp /tmp/libbfpgpu.orig.so paper_1602_04716_b200/libbfpgpu.so
