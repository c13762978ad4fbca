set -x
timeout 300 python -m pytest tests -x -q -m gpu -k "fused" 2>&1 | tail -3
for path in 3 1; do timeout 300 python scripts/bench_press.py 512 512 90 --path $path --reps 3; done
LESB_FUSED_TILE=1 timeout 300 python scripts/bench_press.py 512 512 90 --path 3 --reps 3
timeout 300 python scripts/bench_press.py 150 150 90 --path 3
timeout 600 ncu --set full --clock-control none --import-source on -k regex:k_sor_rbmarch -s 4 -c 1 -o gpurun_out/march512c python scripts/bench_press.py 512 512 90 --path 3 --reps 1 --n-iter 4 > /dev/null 2>&1
