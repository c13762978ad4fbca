for d in 0 1 9 3; do echo "debug=$d"; LESB_RES_DEBUG=$d python scripts/res_trace.py 2>&1 | head -3; done
