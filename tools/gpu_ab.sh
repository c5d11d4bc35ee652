for g in 4 2 3; do HTLR_THIN_G=$g python bench.py --workload cfg3 --steps 5 --warmup 3 --no-cpu-baseline > gpurun_out/b3_$g.json 2>gpurun_out/b3_$g.err; done
