set -x
python scripts/prof_press.py --path 2
python scripts/prof_press.py --path 1
python scripts/prof_press.py 512 512 90 --path 0 --reps 3
timeout 600 ncu --set full --clock-control none --import-source on -k regex:k_sor_resident -s 1 -c 1 -o gpurun_out/prof_resident python scripts/prof_press.py --path 2 --reps 2 > gpurun_out/ncu_res.log 2>&1
timeout 600 ncu --set full --clock-control none --import-source on -k regex:k_sor_rb -s 10 -c 2 -o gpurun_out/prof_rb python scripts/prof_press.py --path 1 --reps 1 --n-iter 10 > gpurun_out/ncu_rb.log 2>&1
timeout 600 ncu --set full --clock-control none --import-source on -k regex:"k_fused_rhs|k_velnw_bondv1|k_press_halo" -s 3 -c 3 -o gpurun_out/prof_stages python bench.py --steps 3 --warmup 3 --no-cpu --no-e2e > gpurun_out/ncu_stages.log 2>&1
ls -la gpurun_out
