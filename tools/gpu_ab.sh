export PYTHONPATH=$PWD
timeout 900 python -m pytest tests/test_gpu_multi.py tests/test_gpu_mapped.py -m gpu -x -q 2>&1 | tail -2 > gpurun_out/ab.log
timeout 600 python tools/shard_graph_probe.py >> gpurun_out/ab.log 2>&1
timeout 600 python tools/shard_probe.py 2>&1 | tail -5 | cut -c1-330 >> gpurun_out/ab.log
HTLR_DIST_BACKEND=gloo timeout 600 python bench.py --gpus 2 --steps 5 --warmup 3 --no-cpu-baseline 2>/dev/null | cut -c1-200 >> gpurun_out/ab.log
