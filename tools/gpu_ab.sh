HTLR_GRAPHS=0 timeout 1800 python -m pytest tests -m gpu -x -q 2>&1 | tail -3
