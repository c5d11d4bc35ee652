for v in 0 1; do HTLR_SPLITK=$v python bench.py --workload cfg2 --steps 20 --warmup 5 --no-cpu-baseline > gpurun_out/b2_$v.json 2>gpurun_out/b2_$v.err; done
