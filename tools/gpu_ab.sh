timeout 1800 python -m pytest tests -m gpu -x -q 2>&1 | tail -2
for w in cfg2 cfg3; do python bench.py --workload $w --steps 10 --warmup 3 > gpurun_out/bench_$w.json 2>gpurun_out/bench_$w.err; done
