set -x
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv
python -m pytest tests -m gpu -x -q 2>&1 | tail -15 > gpurun_out/r02_gpu_tests0.log
python bench.py --steps 3 --warmup 3 > gpurun_out/r02_bench0.json 2> gpurun_out/r02_bench0.err
tail -3 gpurun_out/r02_gpu_tests0.log; cat gpurun_out/r02_bench0.json | head -c 600
