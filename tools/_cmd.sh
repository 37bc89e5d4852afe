timeout 240 python -m pytest tests/test_dist.py -x -q -m gpu > gpurun_out/d.log 2>&1; rc=$?; tail -3 gpurun_out/d.log
if [ $rc -ne 0 ]; then grep -E "^E  " gpurun_out/d.log | grep -v "File\|\^\^" | head -12; exit 1; fi
for n in 2 4; do timeout 150 python -m torch.distributed.run --nnodes=1 --nproc-per-node=$n --master-addr 127.0.0.1 --master-port 295$n$i bench.py --gpus $n --steps 20 --warmup 3 > gpurun_out/b${n}.log 2>&1; done
for f in gpurun_out/b2.log gpurun_out/b4.log; do grep '^{' $f | python -c "import json,sys; d=json.loads(sys.stdin.read()); print(d['n_gpus'], round(d['ms_per_step'],4), round(d['value']/1e6,1), [round(r['sum_ms'],2) for r in d['per_rank']], round(d['e2e']['value']/1e6,1), {k: round(v*1e3,1) for k,v in d['kernel_ms_rank0'].items()})" || tail -3 $f; done
