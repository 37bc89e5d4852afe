# sharded-step device timeline (RS_TRACE=1) at N=2 and N=4.  usage: bash tools/r2_dist_trace.sh TAG
T=${1:-r2t}
for N in 2 4; do
  RS_TRACE=1 timeout 900 python bench.py --gpus $N --steps 10 --warmup 5 > gpurun_out/${T}_trace$N.json 2> gpurun_out/${T}_trace$N.err
  grep "^{" gpurun_out/${T}_trace$N.json | python -c "import json,sys; d=json.loads(sys.stdin.read()); print($N, d['ms_per_step']); [print(' ', k, v) for k, v in d.get('timeline_us_rank0', {}).items()]"
done
