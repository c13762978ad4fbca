set -x
LESB_RESIDENT_GENERIC=1 python scripts/prof_press.py --path 2 --n-iter 1
LESB_RESIDENT_GENERIC=1 python scripts/prof_press.py --path 2 --n-iter 2
LESB_RESIDENT_GENERIC=1 timeout 600 ncu --set full --clock-control none --import-source on -k regex:k_sor -s 1 -c 1 -o gpurun_out/prof_fixed python scripts/prof_press.py --path 2 --reps 2 --n-iter 1 > gpurun_out/ncu_fixed.log 2>&1
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launch_press.csv python scripts/prof_press.py --path 2 --reps 2 --n-iter 1 > /dev/null 2>&1
cat gpurun_out/launch_press.csv | tail -5
