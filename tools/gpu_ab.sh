for v in 0 1; do HTLR_MT224=$v python bench.py --workload cfg3 --steps 5 --warmup 3 --no-cpu-baseline > gpurun_out/b3_$v.json 2>gpurun_out/b3_$v.err; done
HTLR_MT224=1 timeout 900 python -m pytest tests/test_gpu_parity.py -x -q -k "cfg3 or small or random" 2>&1 | tail -2
