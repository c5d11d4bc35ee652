timeout 900 python -m pytest tests/test_gpu_multi.py tests/test_gpu_mapped.py -x -q 2>&1 | tail -2
export HTLR_DIST_BACKEND=gloo
for w in cfg2 cfg5 cfg4; do timeout 900 python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 --master-port $((29500 + RANDOM % 400)) bench.py --gpus 2 --workload $w --steps 3 --warmup 3 --no-cpu-baseline > gpurun_out/multi_$w.json 2> gpurun_out/multi_$w.err; echo "$w rc=$?"; done
