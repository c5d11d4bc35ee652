timeout 1800 python -m pytest tests -m gpu -x -q 2>&1 | tail -2
python -c "import __graft_entry__ as g; g.smoke(); print('smoke ok')" 2>&1 | tail -1
for w in cfg1 cfg2 cfg3 cfg4 cfg5; do python bench.py --workload $w --steps 10 --warmup 3 > gpurun_out/bench_$w.json 2>gpurun_out/bench_$w.err; done
python bench.py --impl reference --steps 3 --warmup 3 > gpurun_out/bench_ref_cfg4.json 2>gpurun_out/bench_ref.err
