# Scratch A/B script shipped to the GPU box with gpurun (dev aid; the content
# changes from experiment to experiment).  Example:
#   gpurun --timeout 1200 -- 'mkdir -p gpurun_out; bash tools/gpu_ab.sh'
for w in cfg2 cfg4; do
  python bench.py --workload $w --steps 10 --warmup 3 --no-cpu-baseline > gpurun_out/b_$w.json 2> gpurun_out/b_$w.err
done
