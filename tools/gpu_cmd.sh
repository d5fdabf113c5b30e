timeout 900 python -m pytest tests -m gpu -x -q -k "prefetch or api" 2>&1 | tail -2
