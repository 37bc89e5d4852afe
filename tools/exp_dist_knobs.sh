# sharded-step knob sweep at N (default 4): ms_per_step per env setting, then the
# device timeline of the last setting.  usage: bash tools/exp_dist_knobs.sh N "ENV1" "ENV2" ...
N=${1:-4}; shift
for E in "$@"; do
  env $E timeout 600 python bench.py --gpus $N --steps 30 --warmup 5 > gpurun_out/knob.json 2> gpurun_out/knob.err
  echo "$E => $(grep '^{' gpurun_out/knob.json | python -c "import json,sys; d=json.loads(sys.stdin.read()); print(round(d['ms_per_step']*1e3,1), 'us; e2e', round(d['e2e']['ms_per_step']*1e3,1), d['step_ms_rank0'])" 2>&1 | tail -1)"
done
E="${@: -1}"
env $E RS_TRACE=1 timeout 600 python bench.py --gpus $N --steps 10 --warmup 5 > gpurun_out/knob_t.json 2> gpurun_out/knob_t.err
grep "^{" gpurun_out/knob_t.json | python -c "import json,sys; d=json.loads(sys.stdin.read()); [print(' ', k, v) for k, v in d.get('timeline_us_rank0', {}).items()]"
