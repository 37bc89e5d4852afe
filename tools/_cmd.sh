timeout 240 python -m pytest tests/test_dist.py -x -q -m gpu > gpurun_out/d.log 2>&1; rc=$?; tail -2 gpurun_out/d.log
if [ $rc -ne 0 ]; then grep -E "^E  " gpurun_out/d.log | grep -v "File\|\^\^" | head -12; exit 1; fi
for n in 2 4; do timeout 150 python -m torch.distributed.run --nnodes=1 --nproc-per-node=$n --master-addr 127.0.0.1 --master-port 2956$n bench.py --gpus $n --steps 20 --warmup 3 > gpurun_out/b${n}.log 2>&1; done
for f in gpurun_out/b2.log gpurun_out/b4.log; do grep "^{" $f | python -c "import json,sys; d=json.loads(sys.stdin.read()); print(d['n_gpus'], round(d['ms_per_step'],4), round(d['value']/1e6,1), round(d['e2e']['value']/1e6,1), d['nvlink']['achieved_gbs'])"; done
