export MASTER_ADDR=127.0.0.1 MASTER_PORT=29555 RANK=0 WORLD_SIZE=1 LOCAL_RANK=0
timeout 300 python bench.py --sharded --steps 5 --warmup 3 --no-cpu-baseline > gpurun_out/sh1.log 2>&1; tail -c 600 gpurun_out/sh1.log
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/sh1_launches.csv python bench.py --sharded --steps 3 --warmup 3 --no-cpu-baseline > gpurun_out/sh1_ncu.log 2>&1; echo ncu rc=$?
