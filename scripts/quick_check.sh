#!/bin/bash
# Parity (GPU tests) then one bench line per large config; used between kernel changes.
mkdir -p gpurun_out/quick
timeout 900 python -m pytest tests -m gpu -x -q ${QUICK_PYTEST_ARGS:---ignore=tests/test_gpu_fullsize.py} > gpurun_out/quick/pytest.log 2>&1; echo "pytest rc=$?"; tail -2 gpurun_out/quick/pytest.log
for c in cfg4 cfg3 cfg5; do
  timeout 600 python bench.py --config $c --steps 100 --no-cpu-baseline --e2e-steps 2 > gpurun_out/quick/$c.json 2> gpurun_out/quick/$c.err
  echo "$c rc=$? $(python -c "import json;d=json.loads(open('gpurun_out/quick/$c.json').read().strip().splitlines()[-1]);print(round(d['ms_per_step'],4),'ms',round(d['roofline']['frac'],3))")"
done
