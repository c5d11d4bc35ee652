# Scratch A/B script shipped to the GPU box with gpurun (dev aid; the content
# changes from experiment to experiment).  Example:
#   gpurun --timeout 1200 -- 'mkdir -p gpurun_out; bash tools/gpu_ab.sh'
export PYTHONPATH=$PWD
python -m pytest tests -m gpu -x -q > gpurun_out/gpu_tests.log 2>&1
python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke.log 2>&1
for w in cfg4 cfg2 cfg3 cfg5 cfg1; do
  python bench.py --workload $w --steps 10 --warmup 3 > gpurun_out/b_$w.json 2> gpurun_out/b_$w.err
done
python bench.py --impl reference --steps 3 --warmup 3 > gpurun_out/b_ref.json 2> gpurun_out/b_ref.err
ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches_cfg4.csv \
  python tools/prof_cmd.py cfg4 1 > gpurun_out/ncu_l.log 2>&1
ncu --set full --clock-control none --import-source on -k regex:sep_block -s 5 -c 1 -f -o gpurun_out/r01_cfg4_sep_leaf \
  python tools/prof_cmd.py cfg4 1 > gpurun_out/ncu_f.log 2>&1
tail -n 3 gpurun_out/gpu_tests.log; cat gpurun_out/smoke.log
