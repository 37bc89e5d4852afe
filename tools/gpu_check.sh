#!/bin/bash
# one GPU round: parity tests, smoke, bench, ncu launch list
set -x
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke.log 2>&1; echo SMOKE $? >> gpurun_out/smoke.log
timeout 500 python -m pytest tests -m gpu -q -x > gpurun_out/pytest_gpu.log 2>&1; echo PYTEST $? >> gpurun_out/pytest_gpu.log
timeout 300 python bench.py --steps 10 --warmup 3 --no-cpu-baseline > gpurun_out/bench.log 2>&1 && \
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches.csv python bench.py --steps 2 --warmup 3 --no-cpu-baseline > /dev/null 2>&1
echo DONE
