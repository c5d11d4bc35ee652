# Scratch A/B script shipped to the GPU box with gpurun (dev aid; the content
# changes from experiment to experiment).  Example:
#   gpurun --timeout 1200 -- 'mkdir -p gpurun_out; bash tools/gpu_ab.sh'
export PYTHONPATH=$PWD
python -m pytest tests/test_gpu_multi.py -x -q > gpurun_out/t.log 2>&1
HTLR_DIST_BACKEND=gloo timeout 600 python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 \
  --master-port 29511 bench.py --gpus 2 --steps 3 --warmup 3 --no-cpu-baseline > gpurun_out/b_w2.json 2> gpurun_out/b_w2.err
python tools/phases.py cfg4 > gpurun_out/ph.log 2>&1
tail -n 3 gpurun_out/t.log; tail -c 300 gpurun_out/b_w2.json; head -3 gpurun_out/ph.log
