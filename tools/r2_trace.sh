# parity + timing + device timeline of the fast step.  usage: bash tools/r2_trace.sh TAG
T=${1:-r2x}
timeout 600 python -m pytest tests/test_gpu_parity.py tests/test_c1_full_step.py -x -q > gpurun_out/${T}_tests.log 2>&1; tail -2 gpurun_out/${T}_tests.log
timeout 300 python tools/exp_flush.py 30 > gpurun_out/${T}_flush.json 2>&1; tail -1 gpurun_out/${T}_flush.json | python -c 'import json,sys; d=json.load(sys.stdin); print("step us", [round(x["median_ms"]*1e3,1) for x in d["dirty"]+d["clean"]])'
timeout 300 python tools/exp_trace.py > gpurun_out/${T}_trace.log 2>&1; tail -1 gpurun_out/${T}_trace.log | python -c '
import json,sys
for k,v in json.loads(sys.stdin.read()).items(): print(k, v)'
