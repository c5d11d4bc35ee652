timeout 1200 python -m pytest tests -m gpu -x -q 2>&1 | tail -2
for v in 0 1; do HTLR_PDL=$v PYTHONPATH=. python tools/quick_time.py cfg1 cfg2 cfg3 cfg4 cfg5; done
