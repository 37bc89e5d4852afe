# bench lines of configs 2-5 (4-GPU box): bash tools/gpu_configs.sh TAG
T=${1:-r03}
p() { grep "^{" $1 | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('$1', d.get('n_gpus'), round(d['ms_per_step']*1e3,2), round(d['value']/1e6,1), (d.get('e2e') or {}).get('value'), d.get('balance'))"; }
timeout 600 python bench.py --config c2 --no-cpu-baseline > gpurun_out/${T}_c2.json 2>/dev/null; p gpurun_out/${T}_c2.json
timeout 600 python bench.py --config c3 --no-cpu-baseline > gpurun_out/${T}_c3.json 2>/dev/null; p gpurun_out/${T}_c3.json
timeout 900 python bench.py --config c4 --no-cpu-baseline > gpurun_out/${T}_c4_1.json 2>/dev/null; p gpurun_out/${T}_c4_1.json
for n in 2 4; do
  timeout 900 python -m torch.distributed.run --nnodes=1 --nproc-per-node=$n --master-addr 127.0.0.1 --master-port 2958$n bench.py --gpus $n --config c4 > gpurun_out/${T}_c4_$n.json 2>/dev/null; p gpurun_out/${T}_c4_$n.json
  timeout 600 python -m torch.distributed.run --nnodes=1 --nproc-per-node=$n --master-addr 127.0.0.1 --master-port 2959$n bench.py --gpus $n --config c5 > gpurun_out/${T}_c5_$n.json 2>/dev/null; p gpurun_out/${T}_c5_$n.json
done
