# Round evidence: tests, bench line, reference arm, scaling-size step lines,
# press-only lines (with the reference's CPU solve beside them), ncu launch
# list and full captures.  Outputs under gpurun_out/ev/.
set -x
mkdir -p gpurun_out/ev
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm,memory.total --format=csv > gpurun_out/ev/gpu.txt
timeout 900 python -m pytest tests -q -m gpu > gpurun_out/ev/pytest_gpu.txt 2>&1; tail -3 gpurun_out/ev/pytest_gpu.txt
python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/ev/smoke.txt 2>&1; cat gpurun_out/ev/smoke.txt
timeout 900 python bench.py > gpurun_out/ev/bench.json 2> gpurun_out/ev/bench.err; cat gpurun_out/ev/bench.json
timeout 600 python bench.py --impl reference --steps 3 --warmup 1 > gpurun_out/ev/bench_ref.json 2>&1; tail -1 gpurun_out/ev/bench_ref.json
rm -f gpurun_out/ev/bench_grids.jsonl
for gr in "300 300 90" "600 600 90"; do timeout 600 python bench.py --grid $gr --steps 40 --warmup 5 --no-cpu 2>/dev/null | tail -1 >> gpurun_out/ev/bench_grids.jsonl; done
rm -f gpurun_out/ev/press.jsonl
for path in 0 1; do timeout 300 python scripts/bench_press.py 150 150 90 --path $path >> gpurun_out/ev/press.jsonl; done
timeout 600 python scripts/bench_press.py 512 512 90 --path 1 --reps 5 --cpu >> gpurun_out/ev/press.jsonl
timeout 300 python scripts/bench_press.py 512 512 90 --path 1 --reps 5 --halo press >> gpurun_out/ev/press.jsonl
timeout 300 python scripts/bench_press.py 512 512 90 --path 3 --reps 3 >> gpurun_out/ev/press.jsonl
timeout 600 python scripts/bench_press.py 512 512 90 --scheme twinned --reps 3 --cpu >> gpurun_out/ev/press.jsonl
python scripts/res_trace.py > gpurun_out/ev/res_trace.txt 2>&1
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none -c 60 --csv --log-file gpurun_out/ev/launches.csv python bench.py --steps 6 --warmup 3 --no-cpu --no-e2e --no-extras > /dev/null 2>&1
timeout 900 ncu --set full --clock-control none --import-source on -k regex:"k_sor_resident|k_fused_rhs|k_velnw_bondv1" -s 3 -c 3 -o gpurun_out/ev/step_full python bench.py --steps 3 --warmup 3 --no-cpu --no-e2e --no-extras > gpurun_out/ev/ncu_step.log 2>&1
timeout 900 ncu --set full --clock-control none --import-source on -k regex:"k_sor_rbt" -s 10 -c 2 -o gpurun_out/ev/rbt512_full python scripts/bench_press.py 512 512 90 --path 1 --reps 1 --n-iter 6 > gpurun_out/ev/ncu_rbt512.log 2>&1
ls -la gpurun_out/ev
