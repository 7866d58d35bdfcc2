# round-2 evidence run, part 1: GPU tests, smoke, bench (both arms)
mkdir -p gpurun_out
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv
timeout 1800 python -m pytest tests -q -m gpu 2>&1 | tail -30 > gpurun_out/r02_gputests.log
tail -3 gpurun_out/r02_gputests.log
python -c "import __graft_entry__ as g; g.smoke()" 2>&1 | tail -2 | tee gpurun_out/r02_smoke.log
timeout 1500 python bench.py --steps 3 --warmup 3 > gpurun_out/r02_bench_c3.json 2> gpurun_out/r02_bench_c3.err
tail -c 400 gpurun_out/r02_bench_c3.json; tail -3 gpurun_out/r02_bench_c3.err
timeout 900 python bench.py --impl reference --steps 2 --warmup 1 > gpurun_out/r02_bench_reference_arm.json 2> gpurun_out/r02_bench_reference_arm.err
tail -c 300 gpurun_out/r02_bench_reference_arm.json
./tools/bench_gemm > gpurun_out/r02_gemm_bench.txt 2>&1; cat gpurun_out/r02_gemm_bench.txt | cut -c1-120
