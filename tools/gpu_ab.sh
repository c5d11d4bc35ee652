timeout 1500 python -m pytest tests/test_gpu_mapped.py tests/test_gpu_blocks_api.py -x -q 2>&1 | tail -2
HTLR_TIMING=1 PYTHONPATH=. python tools/construct_split.py cfg5 cfg4 2>&1 | tail -20
