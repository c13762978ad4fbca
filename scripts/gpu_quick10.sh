set -x
timeout 600 python -m pytest tests -x -q -m gpu 2>&1 | tail -3
for path in 1 3; do timeout 300 python scripts/bench_press.py 512 512 90 --path $path --reps 3; done
timeout 300 python scripts/bench_press.py 512 512 90 --path 1 --reps 3 --halo press
