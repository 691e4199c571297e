set -u
mkdir -p gpurun_out/ncu2 /tmp/ncu
timeout 900 python -m pytest tests/test_gpu_jit.py -q -x > gpurun_out/pytest_jit.log 2>&1; echo jit_rc=$?; tail -2 gpurun_out/pytest_jit.log
for spec in c3_mul:C3:mul c4_mul_8_15:C4:mul_1/8/15 c5:C5:mul_add; do
  IFS=: read name cfg ops <<< "$spec"
  timeout 600 ncu --set full --clock-control none --import-source on -k regex:k_arith -s 0 -c 1 \
    -o /tmp/ncu/$name -f python tools/profile_kernels.py --config $cfg --ops $ops --iters 1 > gpurun_out/ncu2/$name.log 2>&1; echo prof_${name}_rc=$?
  ncu -i /tmp/ncu/$name.ncu-rep --page details > gpurun_out/ncu2/$name.details.txt 2>&1
  ncu -i /tmp/ncu/$name.ncu-rep --page raw --csv > gpurun_out/ncu2/$name.raw.csv 2>&1
done
