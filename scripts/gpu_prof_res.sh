set -x
timeout 600 ncu --set full --clock-control none --import-source on -k regex:k_sor_resident -s 1 -c 1 -o gpurun_out/prof_resident2 python scripts/prof_press.py --path 2 --reps 2 > gpurun_out/ncu_res2.log 2>&1
tail -3 gpurun_out/ncu_res2.log
