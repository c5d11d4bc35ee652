python -m pytest tests/test_gpu_edge.py tests/test_gpu_parity.py -x -q 2>&1 | tail -3
for v in 0 ""; do HTLR_GEMM_NARROW=$v PYTHONPATH=. python tools/quick_time.py cfg2 cfg3 cfg4; done
HTLR_SPLITK=1 PYTHONPATH=. python tools/quick_time.py cfg2 cfg3
python bench.py --workload cfg2 --steps 20 --warmup 5 --no-cpu-baseline > gpurun_out/b2.json 2>gpurun_out/b2.err
python tools/prof_cmd.py cfg2 3 && ncu --metrics gpu__time_duration.sum --clock-control none -s 20 --csv --log-file gpurun_out/launches_cfg2.csv python tools/prof_cmd.py cfg2 3 > gpurun_out/ncu2.log 2>&1
