mkdir -p gpurun_out
timeout 900 python tools/project_c5.py --lead 24 --repeats 1 > gpurun_out/r02_c5_dbg.json 2> gpurun_out/r02_c5_dbg.log
tail -3 gpurun_out/r02_c5_dbg.log | cut -c1-1500
bash tools/r02_s5c.sh
