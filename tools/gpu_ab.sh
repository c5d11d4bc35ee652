python -m pytest tests/test_gpu_mapped.py tests/test_gpu_multi.py -x -q 2>&1 | tail -2
PYTHONPATH=. python tools/quick_time.py cfg5
python bench.py --workload cfg5 --steps 5 --warmup 3 --no-cpu-baseline > gpurun_out/b5.json 2>gpurun_out/b5.err
