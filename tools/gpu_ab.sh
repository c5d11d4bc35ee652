export PYTHONPATH=$PWD
timeout 900 python -m pytest tests/test_gpu_separable.py tests/test_gpu_parity.py -m gpu -x -q 2>&1 | tail -2 > gpurun_out/ab.log
for v in 1 0; do
echo "== HTLR_HALF_PLANES=$v" >> gpurun_out/ab.log
HTLR_HALF_PLANES=$v timeout 300 python tools/phases.py cfg4 50 2>&1 | head -4 >> gpurun_out/ab.log
HTLR_HALF_PLANES=$v timeout 300 python bench.py --steps 50 --warmup 5 --no-cpu-baseline 2>/dev/null | python -c "import sys,json; d=json.loads(sys.stdin.read().strip().splitlines()[-1]); print(d['ms_per_step'], d['e2e']['ms_per_step'])" >> gpurun_out/ab.log
done
