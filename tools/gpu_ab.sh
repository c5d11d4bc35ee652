timeout 1500 python -m pytest tests/test_gpu_edge.py tests/test_gpu_parity.py -x -q 2>&1 | tail -2
for w in cfg4 cfg3 cfg2; do python bench.py --workload $w --steps 5 --warmup 3 --no-cpu-baseline > gpurun_out/b_$w.json 2>gpurun_out/b_$w.err; done
