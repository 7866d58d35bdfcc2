# session-5 call A: GPU tests, bench line, C3 launch list + --set full per kernel class
mkdir -p gpurun_out
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv
timeout 1800 python -m pytest tests -q -m gpu 2>&1 | tail -30 > gpurun_out/r02_gputests.log
tail -5 gpurun_out/r02_gputests.log
timeout 1200 python bench.py --steps 3 --warmup 3 > gpurun_out/r02_bench_c3.json 2> gpurun_out/r02_bench_c3.err
tail -c 600 gpurun_out/r02_bench_c3.json; tail -3 gpurun_out/r02_bench_c3.err
bash tools/r02_ncu.sh
