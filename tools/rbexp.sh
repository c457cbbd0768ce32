python -m pytest tests -m gpu -x -q 2>&1 | tail -4
python tools/kernel_times.py --steps 3 2>&1 | tail -12
python bench.py --steps 20 --warmup 5 2>&1 | tail -1 | head -c 300
