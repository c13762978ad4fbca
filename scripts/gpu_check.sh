# quick GPU check: full parity suite + the press-only lines
set -x
timeout 600 python -m pytest tests -x -q -m gpu 2>&1 | tail -2
timeout 300 python scripts/bench_press.py 512 512 90 --path 1 --reps 3
timeout 300 python scripts/bench_press.py 150 150 90 --path 1
