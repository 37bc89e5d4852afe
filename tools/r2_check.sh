# quick GPU check of the single-GPU step: parity tests, smoke, step time, phase times.  usage: bash tools/r2_check.sh TAG
T=${1:-r2x}
timeout 600 python -m pytest tests/test_gpu_parity.py tests/test_c1_full_step.py -x -q > gpurun_out/${T}_tests.log 2>&1; tail -4 gpurun_out/${T}_tests.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/${T}_smoke.log 2>&1; tail -1 gpurun_out/${T}_smoke.log
timeout 300 python tools/exp_flush.py 30 > gpurun_out/${T}_flush.json 2>&1; tail -1 gpurun_out/${T}_flush.json
RS_NO_GRAPH=1 timeout 300 python tools/exp_phases.py > gpurun_out/${T}_phases.json 2>&1; tail -1 gpurun_out/${T}_phases.json
