for v in 128 256; do HTLR_GEN_MT=$v python bench.py --workload cfg2 --steps 20 --warmup 5 --no-cpu-baseline > gpurun_out/b2_$v.json 2>gpurun_out/b2_$v.err; done
HTLR_GEN_MT=256 timeout 900 python -m pytest tests/test_gpu_parity.py -x -q -k "cfg2 or single" 2>&1 | tail -2
