# The bounds-checked build (-DRS_BOUNDS: every computed index of the fast
# step, the split-kernel finish and the sharded finish range-checked on the
# device) over the parity tests and the sanitizer case -- the substitute for
# compute-sanitizer, which is closed on this pool.  usage: bash tools/checked.sh TAG
T=${1:-r2}
make -s -C paper_2505_12663_b200/csrc -j8 OUT=../_lib/checked/librsgpu.so OBJDIR=../_lib/obj_checked EXTRA=-DRS_BOUNDS ../_lib/checked/librsgpu.so
export RS_LIB_PATH=$PWD/paper_2505_12663_b200/_lib/checked/librsgpu.so
timeout 1200 python -m pytest tests/test_gpu_parity.py tests/test_c1_full_step.py tests/test_dist_local.py -q -x > gpurun_out/${T}_checked_tests.log 2>&1; tail -2 gpurun_out/${T}_checked_tests.log
timeout 600 python tools/sanitize_case.py > gpurun_out/${T}_checked_case.log 2>&1; tail -2 gpurun_out/${T}_checked_case.log
grep -c "bounds" gpurun_out/${T}_checked_tests.log gpurun_out/${T}_checked_case.log
