for d in 0 1 2 3 4 6 7; do echo "debug=$d"; LESB_RES_DEBUG=$d python scripts/prof_press.py --path 2 2>&1 | tail -1; done
