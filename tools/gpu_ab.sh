export PYTHONPATH=$PWD
sed -i 's/^for rule, eta in \[("weak", None)\]:/for rule, eta in [("weak", None), ("strong", 2.0), ("strong", 0.7)]:/' tools/weak_dbg.py
TAG=fixed python tools/weak_dbg.py > gpurun_out/w.log 2>&1
python -m pytest tests/test_gpu_separable.py tests/test_gpu_multi.py -x -q > gpurun_out/t.log 2>&1
cat gpurun_out/w.log; tail -n 2 gpurun_out/t.log
