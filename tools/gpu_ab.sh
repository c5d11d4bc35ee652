export PYTHONPATH=$PWD
timeout 900 python -m pytest tests/test_gpu_separable.py tests/test_gpu_multi.py -m gpu -x -q 2>&1 | tail -2 > gpurun_out/ab.log
timeout 300 python tools/phases.py cfg4 50 >> gpurun_out/ab.log 2>&1
for i in 1 2; do
timeout 300 python bench.py --steps 50 --warmup 5 --no-cpu-baseline 2>/dev/null | python -c "import sys,json; d=json.loads(sys.stdin.read().strip().splitlines()[-1]); print(d['ms_per_step'], d['e2e']['ms_per_step'])" >> gpurun_out/ab.log
done
