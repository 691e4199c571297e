set -x
P="python tools/profile_kernels.py --config C2 --iters 4"
$P > gpurun_out/plain.log 2>&1 && \
ncu --metrics gpu__time_duration.sum --clock-control none -k regex:k_arith --csv --log-file gpurun_out/launches_c2.csv $P > gpurun_out/ncu1.log 2>&1
echo rc1=$?
$P > gpurun_out/plain2.log 2>&1 && \
ncu --set full --clock-control none --import-source on -k regex:k_arith -s 2 -c 2 -o gpurun_out/prof_c2 $P > gpurun_out/ncu2.log 2>&1
echo rc2=$?
ls -la gpurun_out
