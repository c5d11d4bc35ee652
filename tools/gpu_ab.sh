python -m pytest tests -m gpu -x -q 2>&1 | tail -2
for v in 1 2; do HTLR_NARROW_CPS=$v PYTHONPATH=. python tools/quick_time.py cfg1 cfg2 cfg3 cfg4 cfg5; done
python bench.py --workload cfg2 --steps 20 --warmup 5 --no-cpu-baseline > gpurun_out/b2.json 2>gpurun_out/b2.err
