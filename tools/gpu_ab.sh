# A/B: leaf z sweep from u with the upward pass on the side stream; SMs left to the side stream
export PYTHONPATH=$PWD
for cfg in "0 20" "1 48" "1 64" "1 0" "0 20" "1 48" "1 40" "1 56"; do
set -- $cfg
echo "== HTLR_Z_FROM_U=$1 HTLR_LEVEL_SMS=$2" >> gpurun_out/ab.log
HTLR_Z_FROM_U=$1 HTLR_LEVEL_SMS=$2 timeout 300 python bench.py --steps 50 --warmup 5 --no-cpu-baseline 2>/dev/null | python -c "import sys,json; d=json.loads(sys.stdin.read().strip().splitlines()[-1]); print(d['ms_per_step'], d['e2e']['ms_per_step'])" >> gpurun_out/ab.log
done
