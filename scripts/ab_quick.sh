set -e
timeout 600 python -m pytest tests/test_gpu_parity.py tests/test_gpu_slabs.py -q -m gpu -x 2>&1 | tail -2
for r in 1 2 3; do
  timeout 300 python bench.py --steps 200 --warmup 20 2>/dev/null | python -c "import json,sys; d=json.loads(sys.stdin.readlines()[-1]); print(d['value'], d['ms_per_step'], d['roofline']['frac'], d['e2e']['value'])"
done
timeout 300 python scripts/res_trace.py 2>&1 | head -6
