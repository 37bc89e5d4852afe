# round-end evidence: GPU tests, bench lines (N=1,2,4 + reference arm), launch list, one ncu --set full capture
# usage (4-GPU box): bash tools/gpu_final.sh TAG
T=${1:-r03}
set -x
timeout 900 python -m pytest tests -x -q -m gpu > gpurun_out/${T}_gpu.log 2>&1; tail -2 gpurun_out/${T}_gpu.log
timeout 300 python bench.py > gpurun_out/${T}_bench1.json 2> gpurun_out/${T}_bench1.err; tail -c 300 gpurun_out/${T}_bench1.json
timeout 300 python bench.py --impl reference --steps 3 --warmup 3 > gpurun_out/${T}_ref.json 2>&1; tail -c 300 gpurun_out/${T}_ref.json
for n in 2 4; do
  timeout 300 python -m torch.distributed.run --nnodes=1 --nproc-per-node=$n --master-addr 127.0.0.1 --master-port 2957$n bench.py --gpus $n > gpurun_out/${T}_bench$n.json 2>/dev/null; grep "^{" gpurun_out/${T}_bench$n.json | tail -c 300
done
timeout 300 ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv --log-file gpurun_out/${T}_launches.csv python bench.py --steps 2 --warmup 3 --no-cpu-baseline > gpurun_out/${T}_ncu.log 2>&1
RS_NO_GRAPH=1 timeout 600 ncu --set full --import-source on --clock-control none -k "regex:k_fdedup|k_ftable|k_ftile|k_finish" --launch-skip 60 --launch-count 6 -o gpurun_out/${T}_final python bench.py --steps 2 --warmup 3 --no-cpu-baseline > gpurun_out/${T}_ncu_full.log 2>&1
ls -la gpurun_out/ | grep $T
