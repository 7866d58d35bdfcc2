mkdir -p gpurun_out
timeout 900 python tools/project_c5.py --lead 24 --repeats 1 > gpurun_out/r02_c5_dbg.json 2> gpurun_out/r02_c5_dbg.log || { tail -3 gpurun_out/r02_c5_dbg.log | cut -c1-800; exit 1; }
tail -2 gpurun_out/r02_c5_dbg.log | cut -c1-800
timeout 3000 python tools/project_c5.py --lead 24 48 72 > gpurun_out/r02_c5.json 2> gpurun_out/r02_c5.log
tail -c 1500 gpurun_out/r02_c5.json; tail -5 gpurun_out/r02_c5.log | cut -c1-800
