# round-2 evidence pass: GPU suite, smoke, benches of every config (+ reference arm), launch list, ncu --set full, construction
export PYTHONPATH=$PWD
timeout 2400 python -m pytest tests -m gpu -x -q > gpurun_out/g_tests.log 2>&1; echo "rc=$?" >> gpurun_out/g_tests.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/g_smoke.log 2>&1; echo "rc=$?" >> gpurun_out/g_smoke.log
timeout 600 python bench.py --steps 20 --warmup 5 > gpurun_out/g_bench_cfg4.json 2> gpurun_out/g_bench_cfg4.err
timeout 600 python bench.py --impl reference --steps 3 --warmup 1 > gpurun_out/g_bench_ref_cfg4.json 2> gpurun_out/g_bench_ref_cfg4.err
for w in cfg1 cfg2 cfg3 cfg5; do
timeout 600 python bench.py --workload $w --steps 10 --warmup 3 --no-cpu-baseline > gpurun_out/g_bench_$w.json 2> gpurun_out/g_bench_$w.err
done
ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/g_launches_cfg4.csv python tools/prof_cmd.py cfg4 1 > /dev/null 2>&1
timeout 600 ncu --set full --clock-control none --import-source on -k regex:band_plane_kernel -s 3 -c 1 -o gpurun_out/ncu_r02_cfg4_band_plane_kernel python tools/prof_cmd.py cfg4 1 > gpurun_out/g_ncu_plane.log 2>&1
timeout 600 ncu --set full --clock-control none --import-source on -k regex:band_line_kernel -s 2 -c 1 -o gpurun_out/ncu_r02_cfg4_band_line_kernel python tools/prof_cmd.py cfg4 1 > gpurun_out/g_ncu_line.log 2>&1
HTLR_TIMING=1 timeout 300 python tools/construct_time.py cfg4 cfg3 cfg5 cfg2 cfg1 > gpurun_out/g_construct.log 2>&1
timeout 300 python tools/phases.py cfg4 30 > gpurun_out/g_phases_cfg4.log 2>&1
