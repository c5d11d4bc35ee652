export PYTHONPATH=$PWD
for i in 1 2 3 4 5 6; do
timeout 300 python bench.py --steps 20 --warmup 5 --no-cpu-baseline 2>/dev/null | python -c "import sys,json; d=json.loads(sys.stdin.read().strip().splitlines()[-1]); print(d['ms_per_step'], d['e2e']['ms_per_step'], d['e2e']['ms_min'])" >> gpurun_out/ab.log
done
timeout 300 python -m pytest tests/test_gpu_separable.py -m gpu -x -q -k "host or graph or banded_random" 2>&1 | tail -1 >> gpurun_out/ab.log
