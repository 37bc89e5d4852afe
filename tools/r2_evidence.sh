# Round-2 evidence on one B200: GPU tests, smoke, bench lines (ours + reference arm),
# launch list of the bench, ncu --set full of one eager step (flushed + in-context).
# usage: bash tools/r2_evidence.sh TAG
T=${1:-r2}
timeout 1500 python -m pytest tests -q -m gpu > gpurun_out/${T}_gpu.log 2>&1; tail -2 gpurun_out/${T}_gpu.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/${T}_smoke.log 2>&1; tail -1 gpurun_out/${T}_smoke.log
timeout 600 python bench.py --steps 20 --warmup 5 > gpurun_out/${T}_bench1.json 2> gpurun_out/${T}_bench1.err; tail -c 600 gpurun_out/${T}_bench1.json
timeout 600 python bench.py --impl reference --steps 20 --warmup 5 > gpurun_out/${T}_ref1.json 2>&1; tail -c 300 gpurun_out/${T}_ref1.json
timeout 600 python bench.py --steps 2 --warmup 3 --no-cpu-baseline > gpurun_out/${T}_plain_small.json 2>&1 && \
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none -c 600 --csv --log-file gpurun_out/${T}_launches.csv python bench.py --steps 2 --warmup 3 --no-cpu-baseline > gpurun_out/${T}_ncu_launch.log 2>&1
RS_NO_GRAPH=1 timeout 300 python tools/exp_phases.py > gpurun_out/${T}_phases.json 2>&1 && \
RS_NO_GRAPH=1 timeout 900 ncu --set full --import-source on --clock-control none -k "regex:k_fa$|k_fc|k_fh|k_fclean" --launch-skip 30 --launch-count 6 -o gpurun_out/${T}_full python tools/exp_phases.py > gpurun_out/${T}_ncu_full.log 2>&1
RS_NO_GRAPH=1 timeout 300 python tools/exp_phases.py > /dev/null 2>&1 && RS_NO_GRAPH=1 timeout 900 ncu --set full --cache-control none --clock-control none -k "regex:k_fa$|k_fc|k_fh|k_fclean" --launch-skip 30 --launch-count 6 -o gpurun_out/${T}_ctx python tools/exp_phases.py > gpurun_out/${T}_ncu_ctx.log 2>&1
ls gpurun_out | grep ${T}_
