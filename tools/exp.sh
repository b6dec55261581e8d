timeout 1700 python -m pytest tests -m gpu -q -x --durations=15 2>&1 | tail -30
