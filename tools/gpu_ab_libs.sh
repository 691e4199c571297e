# A/B of prebuilt library variants on the GPU box, interleaved round by round
# so clock / power drift hits every variant alike.  Build the variants here
# first (60 s each):
#   BFP_BUILD_TAG=pf0 BFP_EXTRA_NVCC=-DBFP_PREFETCH=0 python -m paper_1602_04716_b200.build --force
# then on the box:
#   TAGS="base pf0" ROUNDS=3 CONFIGS=C5,C4 bash tools/gpu_ab_libs.sh
# tag "base" is the in-tree paper_1602_04716_b200/libbfpgpu.so, others ab/<tag>/libbfpgpu.so.
# Summary (median per kernel and tag): python tools/ab_summary.py gpurun_out/ab_*.jsonl
set -u
mkdir -p gpurun_out
# the tag order rotates every round (a fixed order biases the later variants:
# the box warms and its power-capped clock drifts within a round)
read -r -a TAGA <<< "$TAGS"
NT=${#TAGA[@]}
for r in $(seq 1 ${ROUNDS:-3}); do
  for k in $(seq 0 $((NT - 1))); do
    tag=${TAGA[$(( (k + r - 1) % NT ))]}
    lib=paper_1602_04716_b200/libbfpgpu.so
    [ "$tag" != base ] && lib=ab/$tag/libbfpgpu.so
    BFP_LIB=$PWD/$lib timeout 900 python bench.py --config ${CONFIGS:-C5,C4} --steps ${STEPS:-20} --no-e2e \
      --no-cpu-baseline --no-ncu >> gpurun_out/ab_$tag.jsonl 2>> gpurun_out/ab_$tag.err
    echo "round $r $tag rc=$?"
  done
done
python tools/ab_summary.py gpurun_out/ab_*.jsonl
