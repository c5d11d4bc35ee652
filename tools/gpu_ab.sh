export PYTHONPATH=$PWD
HTLR_TIMING=1 python tools/quick_time.py cfg4 cfg5 cfg3 > gpurun_out/qt.log 2>&1
python -m pytest tests/test_gpu_separable.py tests/test_gpu_parity.py tests/test_gpu_multi.py -x -q > gpurun_out/t.log 2>&1
cat gpurun_out/qt.log | grep -v "^\[htlr timing\]   sep" ; tail -n 2 gpurun_out/t.log
