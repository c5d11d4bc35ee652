set -x
python -m pytest tests -m gpu -x -q 2>&1 | tail -5
for v in 0 1; do HTLR_GEMM_NARROW=$v PYTHONPATH=. python tools/quick_time.py cfg1 cfg2 cfg3 cfg4; done
for v in 0 1; do HTLR_GEMM_NARROW=$v python bench.py --workload cfg2 --steps 20 --warmup 5 --no-cpu-baseline > gpurun_out/b2_$v.json 2>gpurun_out/b2_$v.err; done
python bench.py --workload cfg4 --steps 10 --warmup 3 --no-cpu-baseline > gpurun_out/b4.json 2>gpurun_out/b4.err
