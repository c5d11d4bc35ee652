export PYTHONPATH=$PWD
timeout 900 python -m pytest tests/test_gpu_separable.py -m gpu -x -q -k "host or out_buffer or graph" 2>&1 | tail -2 > gpurun_out/ab.log
timeout 300 python tools/e2e_probe.py cfg4 2>&1 | grep "pinned" >> gpurun_out/ab.log
timeout 300 python tools/e2e_probe.py cfg4 2>&1 | grep "pinned" >> gpurun_out/ab.log
