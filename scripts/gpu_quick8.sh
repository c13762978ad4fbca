set -x
timeout 300 python -m pytest tests -x -q -m gpu -k resident 2>&1 | tail -2
for d in 0 3; do LESB_RES_DEBUG=$d python scripts/res_trace.py 2>&1 | sed -n 2,3p; done
python scripts/prof_press.py --path 2
