#!/bin/bash
# Run one torchrun rank under compute-sanitizer (debugging the sharded step):
#   torchrun --no-python --nproc-per-node 2 tools/san_rank.sh tests/dist_worker.py adam 32
exec /usr/local/cuda/bin/compute-sanitizer --tool memcheck --print-limit 20 \
  --log-file "gpurun_out/san_rank${LOCAL_RANK}.log" python "$@"
