# compute-sanitizer over tools/sanitize_case.py, ONE tool per invocation
# (usage: bash tools/sanitize.sh memcheck|racecheck|synccheck|initcheck TAG)
TOOL=${1:-memcheck}
T=${2:-r2}
timeout 600 python tools/sanitize_case.py > gpurun_out/${T}_san_plain.log 2>&1 && \
timeout 1800 compute-sanitizer --tool $TOOL --print-limit 50 --target-processes all \
  python tools/sanitize_case.py > gpurun_out/${T}_san_${TOOL}.log 2>&1
echo "rc=$?"; tail -4 gpurun_out/${T}_san_${TOOL}.log
