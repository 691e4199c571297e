timeout 600 python -m pytest tests -q -x -m "gpu and not slow" -k "host" > gpurun_out/pytest_gpu.log 2>&1; echo pytest_rc=$?
tail -2 gpurun_out/pytest_gpu.log
for c in 1048576 4194304 16777216; do
BFP_E2E_CHUNK=$c timeout 900 python bench.py --config C2 --steps 20 --warmup 3 --no-cpu-baseline > gpurun_out/bench_e2e$c.log 2>/dev/null
python3 -c "
import json
for l in open('gpurun_out/bench_e2e$c.log'):
    d=json.loads(l); print('chunk=$c', d['value'], d['e2e'])
"
done
