# one bench run (+ optional launch list) on the GPU box; outputs under gpurun_out/
python bench.py --steps 3 --warmup 3 > gpurun_out/r02_bench_c3.json 2> gpurun_out/r02_bench_c3.err
tail -c 3000 gpurun_out/r02_bench_c3.json
tail -5 gpurun_out/r02_bench_c3.err
