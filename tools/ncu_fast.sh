# ncu --set full of the fast step's kernels (eager launches).  usage: bash tools/ncu_fast.sh TAG
T=${1:-r2x}
RS_NO_GRAPH=1 timeout 300 python tools/exp_phases.py > gpurun_out/${T}_phases.json 2>&1 && cat gpurun_out/${T}_phases.json && \
RS_NO_GRAPH=1 timeout 900 ncu --set full --import-source on --clock-control none -k "regex:k_fa$|k_fc|k_fh|k_fclean" --launch-skip 15 --launch-count 5 -o gpurun_out/${T}_fast python tools/exp_phases.py > gpurun_out/${T}_ncu.log 2>&1; tail -2 gpurun_out/${T}_ncu.log
