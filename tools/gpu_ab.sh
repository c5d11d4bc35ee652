timeout 1800 python -m pytest tests -m gpu -x -q 2>&1 | tail -2
PYTHONPATH=. python tools/quick_time.py cfg1 cfg2 cfg3 cfg4 cfg5
for w in cfg1 cfg2 cfg5; do python bench.py --workload $w --steps 20 --warmup 5 --no-cpu-baseline > gpurun_out/b_$w.json 2>gpurun_out/b_$w.err; done
