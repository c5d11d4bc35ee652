export PYTHONPATH=$PWD
python -m pytest tests/test_gpu_separable.py -x -q -k "random" > gpurun_out/t.log 2>&1
HTLR_SEP_BLOCK=0 python -m pytest tests/test_gpu_separable.py -x -q -k "random" >> gpurun_out/t.log 2>&1
cat gpurun_out/t.log | tail -20
