# Scratch A/B script shipped to the GPU box with gpurun (dev aid; the content
# changes from experiment to experiment).  Example:
#   gpurun --timeout 1200 -- 'mkdir -p gpurun_out; bash tools/gpu_ab.sh'
export PYTHONPATH=$PWD
python tools/e2e_probe.py cfg4 2>&1 | grep -E "pinned|h2d" > gpurun_out/e2e.log
HTLR_OVERLAP_SLABS=2 python tools/e2e_probe.py cfg4 2>&1 | grep "pinned in" >> gpurun_out/e2e.log
HTLR_OVERLAP=0 python tools/e2e_probe.py cfg4 2>&1 | grep "pinned in" >> gpurun_out/e2e.log
python -m pytest tests/test_gpu_separable.py -x -q -k "host" > gpurun_out/t.log 2>&1
HTLR_OVERLAP_SLABS=2 python -m pytest tests/test_gpu_separable.py -x -q -k "host" >> gpurun_out/t.log 2>&1
cat gpurun_out/e2e.log; grep passed gpurun_out/t.log
