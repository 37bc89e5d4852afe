# multi-GPU evidence on one box: the sharded step at N=2 and N=4 (bench.py self-launches torchrun),
# the reference arm at N=4, the sharded parity worker at W=4.  usage: bash tools/r2_multi.sh TAG
T=${1:-r2}
timeout 900 python bench.py --gpus 2 --steps 20 --warmup 5 > gpurun_out/${T}_bench2.json 2> gpurun_out/${T}_bench2.err; grep "^{" gpurun_out/${T}_bench2.json | tail -c 400
timeout 900 python bench.py --gpus 4 --steps 20 --warmup 5 > gpurun_out/${T}_bench4.json 2> gpurun_out/${T}_bench4.err; grep "^{" gpurun_out/${T}_bench4.json | tail -c 400
timeout 900 python bench.py --gpus 4 --impl reference --steps 5 --warmup 3 > gpurun_out/${T}_ref4.json 2> gpurun_out/${T}_ref4.err; grep "^{" gpurun_out/${T}_ref4.json | tail -c 300
timeout 900 python -m pytest tests/test_dist.py -q -m gpu > gpurun_out/${T}_dist4.log 2>&1; tail -2 gpurun_out/${T}_dist4.log
