# multi-rank (loopback) GPU tests on one B200
timeout 900 python -m pytest tests/test_multigpu.py -x -q -m gpu 2>&1 | tail -30 > gpurun_out/r02_multigpu.log
cat gpurun_out/r02_multigpu.log
