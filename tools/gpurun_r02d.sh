# ncu --set full of the banded leaf kernels (config 4), launch list, bench
export PYTHONPATH=$PWD
timeout 600 python -m pytest tests/test_gpu_separable.py tests/test_gpu_multi.py -m gpu -x -q > gpurun_out/d_tests.log 2>&1; echo "rc=$?" >> gpurun_out/d_tests.log
timeout 300 python bench.py --steps 20 --warmup 5 --no-cpu-baseline > gpurun_out/d_bench_cfg4.json 2> gpurun_out/d_bench_cfg4.err
timeout 600 ncu --set full --clock-control none --import-source on -k regex:band_plane_kernel -s 3 -c 1 -o gpurun_out/ncu_r02_cfg4_band_plane_kernel python tools/prof_cmd.py cfg4 1 > gpurun_out/d_ncu_plane.log 2>&1
timeout 600 ncu --set full --clock-control none --import-source on -k regex:band_line_kernel -s 2 -c 1 -o gpurun_out/ncu_r02_cfg4_band_line_kernel python tools/prof_cmd.py cfg4 1 > gpurun_out/d_ncu_line.log 2>&1
ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/d_launches_cfg4.csv python tools/prof_cmd.py cfg4 1 > /dev/null 2>&1
