# Final evidence, part B (one B200): ONE ncu --set full of the fast step's kernels
# (eager launches, caches flushed per kernel) after the same command ran clean.
# usage: bash tools/r2_final_b.sh TAG [extra ncu args, e.g. --cache-control none]
T=${1:-r2f}; shift
RS_NO_GRAPH=1 timeout 300 python tools/exp_phases.py > gpurun_out/${T}_phases.json 2>&1 && \
RS_NO_GRAPH=1 timeout 900 ncu --set full --import-source on --clock-control none "$@" -k "regex:k_fa$|k_fc|k_fh|k_fclean" --launch-skip 30 --launch-count 6 -o gpurun_out/${T}_full python tools/exp_phases.py > gpurun_out/${T}_ncu_full.log 2>&1
tail -2 gpurun_out/${T}_ncu_full.log; ls gpurun_out | grep ${T}_
