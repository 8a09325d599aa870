# The GPU suite on libftblas_checked.so: device bounds assertions (-DFTBLAS_CHECKED; a failed one
# prints its site and traps) and the host code under ASan / UBSan -- the stand-in for
# compute-sanitizer, which this pool does not run.  Each test file under its own timeout.
set -x
python -c "import oracle; oracle.build()"
python -c "from paper_2104_00897_b200 import build; build.build(checked=True)"
export FTBLAS_TEST_LIB=libftblas_checked.so
export ASAN_OPTIONS=detect_leaks=0:protect_shadow_gap=0:alloc_dealloc_mismatch=0:detect_odr_violation=0:abort_on_error=1
export UBSAN_OPTIONS=halt_on_error=1:print_stacktrace=1
ASAN=$(gcc -print-file-name=libasan.so)
: > gpurun_out/r2_checked.log
for f in $(ls tests/test_gpu_*.py | grep -v multirank); do
  LD_PRELOAD=$ASAN timeout ${PER_FILE_TIMEOUT:-900} python -m pytest $f -m gpu -q -p no:cacheprovider >> gpurun_out/r2_checked.log 2>&1
  echo "$f rc=$?" | tee -a gpurun_out/r2_checked.log
done
grep -E "passed|failed|FT_CHECK|AddressSanitizer|runtime error|rc=" gpurun_out/r2_checked.log | tail -40
