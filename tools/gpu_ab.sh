# Scratch A/B script shipped to the GPU box with gpurun (dev aid; the content
# changes from experiment to experiment).  Example:
#   gpurun --timeout 1200 -- 'mkdir -p gpurun_out; bash tools/gpu_ab.sh'
export PYTHONPATH=$PWD
HTLR_TIMING=1 python tools/phases.py cfg4 > gpurun_out/ph.log 2>&1
python tools/quick_time.py cfg4 cfg4 >> gpurun_out/ph.log 2>&1
python -m pytest tests/test_gpu_separable.py tests/test_gpu_multi.py -x -q > gpurun_out/t.log 2>&1
cat gpurun_out/ph.log; tail -n 2 gpurun_out/t.log
