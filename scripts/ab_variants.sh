#!/bin/bash
# A/B of scratch/<name>.so builds: bench.py steps/s and the phase split, alternating, 3 rounds
for r in 1 2 3; do
  for v in "$@"; do
    LESB_LIB=scratch/$v.so timeout 300 python bench.py --steps 200 --warmup 20 --no-cpu 2>/dev/null | python -c "import json,sys; d=json.loads(sys.stdin.readlines()[-1]); ph=d['phase_ms']; print('$v', round(d['value'],1), round(d['ms_per_step'],4), ' '.join('%s=%.1f' % (k[:8], 1e3*v) for k, v in ph.items()))"
  done
done
