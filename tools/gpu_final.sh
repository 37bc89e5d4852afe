# round-end evidence: GPU tests, bench lines, launch list, one ncu --set full capture
set -x
timeout 900 python -m pytest tests -x -q -m gpu > gpurun_out/final_gpu.log 2>&1; tail -2 gpurun_out/final_gpu.log
timeout 300 python bench.py > gpurun_out/final_bench.json 2> gpurun_out/final_bench.err; tail -c 300 gpurun_out/final_bench.json
timeout 300 python bench.py --impl reference --steps 3 --warmup 3 > gpurun_out/final_ref.json 2>&1; tail -c 300 gpurun_out/final_ref.json
timeout 300 python -m torch.distributed.run --nnodes=1 --nproc-per-node=2 --master-addr 127.0.0.1 --master-port 29577 bench.py --gpus 2 > gpurun_out/final_b2.json 2>/dev/null; grep "^{" gpurun_out/final_b2.json | tail -c 300
timeout 300 ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv --log-file gpurun_out/final_launches.csv python bench.py --steps 2 --warmup 3 --no-cpu-baseline > gpurun_out/final_ncu.log 2>&1
RS_NO_GRAPH=1 timeout 600 ncu --set full --import-source on --clock-control none -k "regex:k_fdedup|k_ftable|k_ftile|k_finish" --launch-skip 60 --launch-count 6 -o gpurun_out/r02_final python bench.py --steps 2 --warmup 3 --no-cpu-baseline > gpurun_out/ncu_final.log 2>&1
ls -la gpurun_out/
