# Scratch A/B script shipped to the GPU box with gpurun (dev aid; the content
# changes from experiment to experiment).  Example:
#   gpurun --timeout 1200 -- 'mkdir -p gpurun_out; bash tools/gpu_ab.sh'
export PYTHONPATH=$PWD
python bench.py --workload cfg4 --steps 10 --warmup 3 --no-cpu-baseline > gpurun_out/b_cfg4.json 2> gpurun_out/b_cfg4.err
HTLR_DIST_BACKEND=gloo timeout 600 python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 \
  --master-port 29511 bench.py --gpus 2 --steps 3 --warmup 3 --no-cpu-baseline > gpurun_out/b_cfg4_w2gloo.json 2> gpurun_out/b_cfg4_w2gloo.err
python -m pytest tests/test_gpu_separable.py -q -k "out_buffer" > gpurun_out/t.log 2>&1
tail -n 2 gpurun_out/t.log
