timeout 1500 python -m pytest tests -m gpu -x -q 2>&1 | tail -2
python -c "import __graft_entry__ as g; g.smoke(); print('smoke ok')" 2>&1 | tail -1
for w in cfg1 cfg2 cfg3 cfg4 cfg5; do python bench.py --workload $w --steps 10 --warmup 3 > gpurun_out/bench_$w.json 2>gpurun_out/bench_$w.err; done
python bench.py --impl reference --steps 3 --warmup 3 > gpurun_out/bench_ref_cfg4.json 2>gpurun_out/bench_ref.err
python tools/prof_cmd.py cfg2 1 && ncu --set full --clock-control none --import-source on -k regex:gemm_persistent -s 1 -c 1 -o gpurun_out/r01_cfg2_leaf_gen python tools/prof_cmd.py cfg2 1 > gpurun_out/ncu_a.log 2>&1
