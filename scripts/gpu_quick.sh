# quick GPU check: parity tests + press timing + bench (no e2e/cpu)
set -x
timeout 900 python -m pytest tests -x -q -m gpu 2>&1 | tail -15
python scripts/prof_press.py --path 2
python scripts/prof_press.py --path 1
python scripts/prof_press.py 512 512 90 --path 0 --reps 3
timeout 600 python bench.py --steps 40 --warmup 5 --no-cpu
