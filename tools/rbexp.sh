python -m pytest tests -m gpu -x -q 2>&1 | tail -2
python tools/kernel_times.py --steps 3 2>&1 | grep -E "scatter|combine|total"
