set -x
timeout 300 python -m pytest tests -x -q -m gpu 2>&1 | tail -2
python scripts/res_trace.py
python scripts/prof_press.py --path 2
