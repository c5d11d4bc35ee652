python -m pytest tests/test_gpu_edge.py tests/test_gpu_parity.py -x -q 2>&1 | tail -2
python bench.py --workload cfg3 --steps 5 --warmup 3 --no-cpu-baseline > gpurun_out/b3.json 2>gpurun_out/b3.err
python bench.py --workload cfg2 --steps 10 --warmup 3 --no-cpu-baseline > gpurun_out/b2.json 2>gpurun_out/b2.err
