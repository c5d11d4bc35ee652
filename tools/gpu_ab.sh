# Scratch A/B script shipped to the GPU box with gpurun (dev aid; the content
# changes from experiment to experiment).  Example:
#   gpurun --timeout 1200 -- 'mkdir -p gpurun_out; bash tools/gpu_ab.sh'
export PYTHONPATH=$PWD
for w in cfg1 cfg2 cfg3 cfg4; do
  python tools/phases.py $w 20 2>&1 | head -1 >> gpurun_out/ab.log
  HTLR_CONCURRENT=0 python tools/phases.py $w 20 2>&1 | head -1 | sed 's/^/serial /' >> gpurun_out/ab.log
done
python -m pytest tests/test_gpu_parity.py tests/test_gpu_edge.py -x -q > gpurun_out/t.log 2>&1
cat gpurun_out/ab.log; tail -n 2 gpurun_out/t.log
