timeout 900 python -m pytest tests/test_gpu_integration_stub.py -x -q 2>&1 | tail -5
python bench.py --workload cfg5 --steps 3 --warmup 3 --no-cpu-baseline 2>/dev/null | tail -1 | python -c "import json,sys; d=json.loads(sys.stdin.read()); print(d['construction'], d['config']['l2'])"
