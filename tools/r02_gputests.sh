# full GPU test suite on one B200
timeout 1500 python -m pytest tests -q -m gpu 2>&1 | tail -30 > gpurun_out/r02_gputests.log
cat gpurun_out/r02_gputests.log
