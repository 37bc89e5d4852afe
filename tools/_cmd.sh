timeout 300 python -m pytest tests/test_dist.py -x -q -m gpu > gpurun_out/d.log 2>&1; tail -3 gpurun_out/d.log
for i in 1 2; do timeout 300 python -m torch.distributed.run --nnodes=1 --nproc-per-node=2 --master-addr 127.0.0.1 --master-port 2954$i bench.py --gpus 2 --steps 20 --warmup 3 > gpurun_out/bench2_$i.log 2>&1; done
timeout 300 python bench.py --sharded --steps 10 --warmup 3 > gpurun_out/bench1s.log 2>&1
timeout 300 ncu --metrics gpu__time_duration.sum --clock-control none -c 300 --csv --log-file gpurun_out/launches_s1.csv python bench.py --sharded --steps 2 --warmup 3 > gpurun_out/ncu_s1.log 2>&1
for f in gpurun_out/bench2_1.log gpurun_out/bench2_2.log gpurun_out/bench1s.log; do grep '^{' $f | python -c "import json,sys; d=json.loads(sys.stdin.read()); print(d['n_gpus'], d['ms_per_step'], d['value']/1e6, d.get('table_host_syncs_rank0'), {k: round(v*1e3,1) for k,v in d['kernel_ms_rank0'].items()})"; done
