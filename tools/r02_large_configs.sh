# session-5 call N: MLE protocol at C3, C5 leading blocks and C4 TLR(1e-9) with the final code
python -c "import __graft_entry__ as g; g.smoke()" 2>&1 | tail -2
mkdir -p gpurun_out
timeout 900 python tools/run_mle.py C3 > gpurun_out/r02_mle_c3.json 2> gpurun_out/r02_mle_c3.log
tail -c 700 gpurun_out/r02_mle_c3.json; tail -2 gpurun_out/r02_mle_c3.log | cut -c1-300
timeout 1500 python tools/project_c5.py --lead 24 48 72 > gpurun_out/r02_c5.json 2> gpurun_out/r02_c5.log
tail -c 900 gpurun_out/r02_c5.json
timeout 2400 python tools/run_c4.py --lead 77 --accs 1e-9 > gpurun_out/r02_c4_final.json 2> gpurun_out/r02_c4_final.log
tail -c 1500 gpurun_out/r02_c4_final.json; tail -3 gpurun_out/r02_c4_final.log | cut -c1-300
