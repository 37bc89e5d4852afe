# Final evidence, part A (one B200): GPU tests, smoke, bench lines (ours + reference arm),
# config 3, then ONE ncu: the bench's launch list.  usage: bash tools/r2_final_a.sh TAG
T=${1:-r2f}
timeout 1500 python -m pytest tests -q -m gpu > gpurun_out/${T}_gpu.log 2>&1; tail -2 gpurun_out/${T}_gpu.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/${T}_smoke.log 2>&1; tail -1 gpurun_out/${T}_smoke.log
timeout 600 python bench.py --steps 20 --warmup 5 > gpurun_out/${T}_bench1.json 2> gpurun_out/${T}_bench1.err; tail -c 300 gpurun_out/${T}_bench1.json
timeout 600 python bench.py --impl reference --steps 20 --warmup 5 > gpurun_out/${T}_ref1.json 2>&1; tail -c 200 gpurun_out/${T}_ref1.json
timeout 600 python bench.py --config c3 --steps 30 --warmup 3 > gpurun_out/${T}_c3.json 2>&1; tail -c 200 gpurun_out/${T}_c3.json
timeout 600 python bench.py --steps 2 --warmup 3 --no-cpu-baseline > gpurun_out/${T}_plain_small.json 2>&1 && \
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none -c 600 --csv --log-file gpurun_out/${T}_launches.csv python bench.py --steps 2 --warmup 3 --no-cpu-baseline > gpurun_out/${T}_ncu_launch.log 2>&1
echo done
