# shard probes (emulated worlds), new analytic-plan GPU test, 2-rank gloo harness
export PYTHONPATH=$PWD
timeout 900 python -m pytest tests/test_gpu_separable.py -m gpu -x -q -k "analytic" > gpurun_out/f_tests.log 2>&1; echo "rc=$?" >> gpurun_out/f_tests.log
timeout 600 python tools/shard_graph_probe.py > gpurun_out/f_shard_graph.jsonl 2> gpurun_out/f_shard_graph.err
timeout 600 python tools/shard_probe.py > gpurun_out/f_shard_probe.log 2>&1
HTLR_DIST_BACKEND=gloo timeout 600 python bench.py --gpus 2 --steps 5 --warmup 3 --no-cpu-baseline > gpurun_out/f_bench_gloo2.json 2> gpurun_out/f_bench_gloo2.err
