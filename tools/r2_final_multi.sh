# Final bench lines on one 4xB200 box (no profiler): config 1 at N = 1 / 2 / 4 (+ the reference arm at
# N = 1 and 4), config 3, config 4 at N = 1 / 2 / 4, the W = 4 parity worker.  usage: bash tools/r2_final_multi.sh TAG
T=${1:-r2z}
timeout 600 python bench.py --steps 20 --warmup 5 > gpurun_out/${T}_c1_1.json 2> gpurun_out/${T}_c1_1.err
timeout 600 python bench.py --impl reference --steps 20 --warmup 5 > gpurun_out/${T}_ref1.json 2>&1
for N in 2 4; do timeout 900 python bench.py --gpus $N --steps 30 --warmup 5 > gpurun_out/${T}_c1_$N.json 2> gpurun_out/${T}_c1_$N.err; done
timeout 900 python bench.py --gpus 4 --impl reference --steps 5 --warmup 3 > gpurun_out/${T}_ref4.json 2>&1
timeout 600 python bench.py --config c3 --steps 30 --warmup 3 > gpurun_out/${T}_c3.json 2> gpurun_out/${T}_c3.err
timeout 900 python bench.py --config c4 --steps 10 --warmup 3 > gpurun_out/${T}_c4_1.json 2> gpurun_out/${T}_c4_1.err
for N in 2 4; do timeout 900 python bench.py --gpus $N --config c4 --steps 10 --warmup 3 > gpurun_out/${T}_c4_$N.json 2> gpurun_out/${T}_c4_$N.err; done
timeout 900 python -m pytest tests/test_dist.py -q -m gpu > gpurun_out/${T}_dist4.log 2>&1; tail -1 gpurun_out/${T}_dist4.log
ls gpurun_out | grep ${T}_ | wc -l
