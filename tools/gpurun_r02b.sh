# round-2 profiling pass: launch lists, ncu --set full of the cfg4 kernels, construction split
export PYTHONPATH=$PWD
for w in cfg4 cfg2 cfg1; do
ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches_$w.csv python tools/prof_cmd.py $w 1 > gpurun_out/ncu_l_$w.log 2>&1
done
for k in band_plane_kernel band_line_kernel upward8 downward8; do
timeout 600 ncu --set full --clock-control none --import-source on -k regex:$k -s 2 -c 1 -o gpurun_out/ncu_cfg4_$k python tools/prof_cmd.py cfg4 1 > gpurun_out/ncu_f_$k.log 2>&1
done
timeout 600 ncu --set full --clock-control none --import-source on -k regex:gemm -s 4 -c 2 -o gpurun_out/ncu_cfg2_gemm python tools/prof_cmd.py cfg2 1 > gpurun_out/ncu_f_cfg2.log 2>&1
HTLR_TIMING=1 python tools/construct_split.py cfg4 cfg5 cfg2 > gpurun_out/construct_split.log 2>&1
