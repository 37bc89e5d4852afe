# A/B of env settings on bench.py at N GPUs (ms per step mean / median).  usage: bash tools/exp_ab.sh N "ENV1" "ENV2" ...
N=${1:-1}; shift
for E in "$@"; do
  env $E timeout 600 python bench.py --gpus $N --steps 30 --warmup 5 > gpurun_out/ab.json 2> gpurun_out/ab.err
  echo "N=$N $E => $(grep '^{' gpurun_out/ab.json | python -c "import json,sys; d=json.loads(sys.stdin.read()); print(round(d['ms_per_step']*1e3,1), 'us; med', round(d.get('step_ms_rank0', {}).get('median', 0)*1e3,1), 'e2e', d['e2e'].get('ms_per_step'))" 2>&1 | tail -1)"
done
