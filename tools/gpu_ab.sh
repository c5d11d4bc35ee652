python -m pytest tests/test_gpu_edge.py -x -q 2>&1 | tail -2
for v in 1 2; do HTLR_THIN_TN=$v python bench.py --workload cfg3 --steps 5 --warmup 3 --no-cpu-baseline > gpurun_out/b3_$v.json 2>gpurun_out/b3_$v.err; done
