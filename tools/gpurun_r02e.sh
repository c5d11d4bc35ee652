# whole GPU suite + construction split + cfg4 bench after the analytic banded levels
export PYTHONPATH=$PWD
timeout 2400 python -m pytest tests -m gpu -x -q > gpurun_out/e_tests.log 2>&1; echo "rc=$?" >> gpurun_out/e_tests.log
HTLR_TIMING=1 timeout 300 python tools/construct_time.py cfg4 cfg3 cfg5 > gpurun_out/e_construct.log 2>&1
timeout 300 python bench.py --steps 20 --warmup 5 --no-cpu-baseline > gpurun_out/e_bench_cfg4.json 2> gpurun_out/e_bench_cfg4.err
