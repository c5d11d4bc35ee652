export PYTHONPATH=$PWD
export HTLR_GRAPHS=0
timeout 900 compute-sanitizer --tool memcheck --print-limit 20 python tools/sanitize_small.py > gpurun_out/memcheck.log 2>&1
timeout 900 compute-sanitizer --tool racecheck --racecheck-report hazard --print-limit 20 python tools/sanitize_small.py > gpurun_out/racecheck.log 2>&1
timeout 900 compute-sanitizer --tool synccheck --print-limit 20 python tools/sanitize_small.py > gpurun_out/synccheck.log 2>&1
tail -n 4 gpurun_out/memcheck.log gpurun_out/racecheck.log gpurun_out/synccheck.log
