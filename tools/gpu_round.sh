timeout 900 python -m torch.distributed.run --nnodes=1 --nproc-per-node 1 --master-addr 127.0.0.1 --master-port 29533 bench.py --gpus 1 --steps 20 --warmup 3 --no-cpu-baseline > gpurun_out/torchrun.log 2> gpurun_out/torchrun.err; echo torchrun_rc=$?
cut -c1-300 gpurun_out/torchrun.log; tail -3 gpurun_out/torchrun.err
timeout 600 python -m torch.distributed.run --nnodes=1 --nproc-per-node 1 --master-addr 127.0.0.1 --master-port 29534 bench.py --impl reference --gpus 1 --steps 3 --warmup 3 > gpurun_out/torchrun_ref.log 2>&1; echo ref_rc=$?
cut -c1-200 gpurun_out/torchrun_ref.log
python -c "import __graft_entry__ as g; g.smoke()"; echo smoke_rc=$?
