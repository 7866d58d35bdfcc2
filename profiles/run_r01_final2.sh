#!/bin/bash
# End-of-round verification: GPU tests, smoke, bench line (C2), small outputs.
mkdir -p gpurun_out
python -m pytest tests -m gpu -q > gpurun_out/f2_pytest.log 2>&1; echo "pytest rc $?" >> gpurun_out/f2_pytest.log
python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/f2_smoke.log 2>&1
python bench.py > gpurun_out/f2_bench.json 2> gpurun_out/f2_bench.err
tail -n3 gpurun_out/f2_pytest.log; cat gpurun_out/f2_smoke.log
python -c "import json; d=json.load(open('gpurun_out/f2_bench.json')); print(d['value'], d['e2e']['value'], d['roofline']['frac'], d['roofline']['traffic'], d['step_roofline']['frac'])"
