python -m pytest tests -m gpu -x -q 2>&1 | tail -3
for w in cfg2 cfg5; do python bench.py --workload $w --steps 10 --warmup 3 > gpurun_out/bench_$w.json 2>gpurun_out/bench_$w.err; done
