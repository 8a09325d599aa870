python -c "import oracle; oracle.build()"
python -c "from paper_2104_00897_b200 import build; build.build(checked=True)"
export FTBLAS_TEST_LIB=libftblas_checked.so
export ASAN_OPTIONS=detect_leaks=0:protect_shadow_gap=0:alloc_dealloc_mismatch=0:detect_odr_violation=0:abort_on_error=1
export UBSAN_OPTIONS=halt_on_error=1:print_stacktrace=1
ASAN=$(gcc -print-file-name=libasan.so)
LD_PRELOAD=$ASAN timeout 300 python -m pytest tests/test_gpu_fuzz.py tests/test_gpu_parity.py -m gpu -x -q -s -p no:cacheprovider > gpurun_out/chk1.log 2>&1; echo rc=$?
tail -60 gpurun_out/chk1.log | grep -v "site-packages"
