set -x
timeout 300 python -m pytest tests -x -q -m gpu 2>&1 | tail -3
python scripts/prof_press.py --path 3; python scripts/prof_press.py 512 512 90 --path 3 --reps 3
timeout 600 ncu --set full --clock-control none --import-source on -k regex:k_sor_rbfused -s 3 -c 1 -o gpurun_out/prof_fused3 python scripts/prof_press.py --path 3 --reps 2 > gpurun_out/ncu_fz3.log 2>&1
timeout 600 ncu --set full --clock-control none --import-source on -k regex:k_sor_rbfused -s 3 -c 1 -o gpurun_out/prof_fused512b python scripts/prof_press.py 512 512 90 --path 3 --reps 1 --n-iter 4 > gpurun_out/ncu_fz512b.log 2>&1
