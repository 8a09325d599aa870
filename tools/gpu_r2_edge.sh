set -x
python -c "import oracle; oracle.build()"
timeout 1200 python -m pytest tests/test_gpu_edge.py tests/test_gpu_dmr.py tests/test_abi.py -q -p no:cacheprovider > gpurun_out/r2_edge.log 2>&1; echo pytest_rc=$?
tail -40 gpurun_out/r2_edge.log
