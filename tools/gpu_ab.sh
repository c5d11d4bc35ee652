export PYTHONPATH=$PWD
for w in cfg4 cfg2; do
HTLR_DIST_BACKEND=gloo timeout 600 python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 \
  --master-port 29511 bench.py --workload $w --gpus 2 --steps 3 --warmup 3 --no-cpu-baseline > gpurun_out/b_w2_$w.json 2> gpurun_out/b_w2_$w.err
tail -c 250 gpurun_out/b_w2_$w.json
done
