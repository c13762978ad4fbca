set -x
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm,memory.total --format=csv
python -c "import torch;p=torch.cuda.get_device_properties(0);print(p, p.L2_cache_size)"
timeout 900 python -m pytest tests -x -q -m gpu 2>&1 | tail -30 > gpurun_out/pytest_gpu.log
tail -5 gpurun_out/pytest_gpu.log
timeout 600 python bench.py --steps 40 --warmup 5 > gpurun_out/bench1.json 2> gpurun_out/bench1.err
cat gpurun_out/bench1.json; tail -5 gpurun_out/bench1.err
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv --log-file gpurun_out/launches1.csv python bench.py --steps 4 --warmup 3 --no-cpu --no-e2e > gpurun_out/ncu_bench.log 2>&1
tail -3 gpurun_out/ncu_bench.log
