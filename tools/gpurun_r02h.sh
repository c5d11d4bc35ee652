# round-2 final evidence pass (after the direct-f matvec and the plan split): benches of every config (+ reference arm),
# launch list, ncu --set full of the two banded leaf kernels, phases, construction
export PYTHONPATH=$PWD
timeout 600 python bench.py --steps 20 --warmup 5 > gpurun_out/h_bench_cfg4.json 2> gpurun_out/h_bench_cfg4.err
timeout 600 python bench.py --impl reference --steps 3 --warmup 1 > gpurun_out/h_bench_ref_cfg4.json 2> gpurun_out/h_bench_ref_cfg4.err
for w in cfg1 cfg2 cfg3 cfg5; do
timeout 600 python bench.py --workload $w --steps 10 --warmup 3 --no-cpu-baseline > gpurun_out/h_bench_$w.json 2> gpurun_out/h_bench_$w.err
done
for i in 1 2 3; do timeout 300 python bench.py --steps 20 --warmup 5 --no-cpu-baseline 2>/dev/null | python -c "import sys,json; d=json.loads(sys.stdin.read()); print(d['ms_per_step'], d['e2e']['ms_per_step'], d['e2e'].get('ms_min'))"; done > gpurun_out/h_bench_cfg4_repeats.log 2>&1
ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/h_launches_cfg4.csv python tools/prof_cmd.py cfg4 1 > /dev/null 2>&1
timeout 600 ncu --set full --clock-control none --import-source on -k regex:band_plane_kernel -s 3 -c 1 -o gpurun_out/ncu_r02h_cfg4_band_plane_kernel python tools/prof_cmd.py cfg4 1 > gpurun_out/h_ncu_plane.log 2>&1
timeout 600 ncu --set full --clock-control none --import-source on -k regex:band_line_kernel -s 2 -c 1 -o gpurun_out/ncu_r02h_cfg4_band_line_kernel python tools/prof_cmd.py cfg4 1 > gpurun_out/h_ncu_line.log 2>&1
timeout 600 ncu --set full --clock-control none --import-source on -k regex:downward_cube_kernel -s 2 -c 1 -o gpurun_out/ncu_r02h_cfg4_downward_cube_kernel python tools/prof_cmd.py cfg4 1 > gpurun_out/h_ncu_down.log 2>&1
HTLR_TIMING=1 timeout 300 python tools/construct_time.py cfg4 cfg3 cfg5 cfg2 cfg1 > gpurun_out/h_construct.log 2>&1
timeout 300 python tools/phases.py cfg4 30 > gpurun_out/h_phases_cfg4.log 2>&1
timeout 300 python tools/fdirect_ab.py cfg4 > gpurun_out/h_fdirect_ab.log 2>&1
