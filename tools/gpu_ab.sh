# Scratch A/B script shipped to the GPU box with gpurun (dev aid; the content
# changes from experiment to experiment).  Example:
#   gpurun --timeout 1200 -- 'mkdir -p gpurun_out; bash tools/gpu_ab.sh'
export PYTHONPATH=$PWD
python tools/e2e_probe.py cfg4 > gpurun_out/e2e.log 2>&1
python bench.py --workload cfg4 --steps 10 --warmup 3 > gpurun_out/b_cfg4.json 2> gpurun_out/b_cfg4.err
ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches_cfg4.csv \
  python tools/prof_cmd.py cfg4 1 > gpurun_out/ncu_l.log 2>&1
ncu --set full --clock-control none --import-source on -k regex:sep_block -s 5 -c 1 -f -o gpurun_out/r01_cfg4_sep_leaf \
  python tools/prof_cmd.py cfg4 1 > gpurun_out/ncu_f.log 2>&1
cat gpurun_out/e2e.log
