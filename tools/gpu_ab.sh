export PYTHONPATH=$PWD
timeout 900 python -m pytest tests/test_gpu_separable.py tests/test_gpu_multi.py -m gpu -x -q 2>&1 | tail -2 > gpurun_out/ab.log
timeout 300 python tools/phases.py cfg4 50 >> gpurun_out/ab.log 2>&1
timeout 300 python bench.py --steps 50 --warmup 5 --no-cpu-baseline 2>/dev/null | python -c "import sys,json; d=json.loads(sys.stdin.read().strip().splitlines()[-1]); print(d['ms_per_step'], d['e2e']['ms_per_step'])" >> gpurun_out/ab.log
ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/ab_launches.csv python tools/prof_cmd.py cfg4 1 > /dev/null 2>&1
grep -E "band_line_kernel|band_plane_kernel|cube" gpurun_out/ab_launches.csv | awk -F'","' '{print substr($5,1,70), $NF}' | tail -7 >> gpurun_out/ab.log
