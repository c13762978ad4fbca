set -x
timeout 300 python -m pytest tests -x -q -m gpu 2>&1 | tail -2
python scripts/prof_press.py --path 2 --n-iter 1
python scripts/prof_press.py --path 2
timeout 300 python bench.py --steps 24 --warmup 4 --no-cpu --no-e2e
