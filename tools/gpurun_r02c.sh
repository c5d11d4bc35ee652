# round-2 state check: whole GPU suite, smoke, cfg4 bench (+reference arm), launch list, phases
export PYTHONPATH=$PWD
timeout 2400 python -m pytest tests -m gpu -x -q > gpurun_out/c_tests.log 2>&1; echo "rc=$?" >> gpurun_out/c_tests.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/c_smoke.log 2>&1; echo "rc=$?" >> gpurun_out/c_smoke.log
timeout 600 python bench.py --steps 20 --warmup 5 > gpurun_out/c_bench_cfg4.json 2> gpurun_out/c_bench_cfg4.err
timeout 600 python bench.py --impl reference --steps 3 --warmup 1 > gpurun_out/c_bench_ref_cfg4.json 2> gpurun_out/c_bench_ref_cfg4.err
ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/c_launches_cfg4.csv python tools/prof_cmd.py cfg4 1 > /dev/null 2>&1
timeout 300 python tools/phases.py cfg4 20 > gpurun_out/c_phases_cfg4.log 2>&1
for w in cfg1 cfg2 cfg3 cfg5; do
timeout 600 python bench.py --workload $w --steps 10 --warmup 3 --no-cpu-baseline > gpurun_out/c_bench_$w.json 2> gpurun_out/c_bench_$w.err
done
