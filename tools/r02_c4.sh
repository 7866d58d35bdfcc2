# C4 resolution runs (tools/run_c4.py)
timeout 2400 python tools/run_c4.py --lead 77 100 > gpurun_out/r02_c4.json 2> gpurun_out/r02_c4.log
tail -c 2000 gpurun_out/r02_c4.log
