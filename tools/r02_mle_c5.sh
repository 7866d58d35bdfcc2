# final-tree reruns: MLE protocol at C3, C5 leading blocks
mkdir -p gpurun_out
timeout 900 python tools/run_mle.py C3 > gpurun_out/r02_mle_c3.json 2> gpurun_out/r02_mle_c3.log
tail -c 500 gpurun_out/r02_mle_c3.json
timeout 1500 python tools/project_c5.py --lead 24 48 72 > gpurun_out/r02_c5.json 2> gpurun_out/r02_c5.log
tail -c 900 gpurun_out/r02_c5.json
