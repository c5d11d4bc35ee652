# quick GPU check: separable/banded parity tests, smoke, cfg4 bench + launch list
export PYTHONPATH=$PWD
timeout 900 python -m pytest tests/test_gpu_separable.py tests/test_gpu_parity.py tests/test_gpu_multi.py -m gpu -x -q > gpurun_out/q_tests.log 2>&1; echo "rc=$?" >> gpurun_out/q_tests.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/q_smoke.log 2>&1; echo "rc=$?" >> gpurun_out/q_smoke.log
timeout 300 python bench.py --steps 20 --warmup 5 --no-cpu-baseline > gpurun_out/q_bench_cfg4.json 2> gpurun_out/q_bench_cfg4.err
ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/q_launches_cfg4.csv python tools/prof_cmd.py cfg4 1 > /dev/null 2>&1
timeout 300 python tools/phases.py cfg4 20 > gpurun_out/q_phases_cfg4.log 2>&1
