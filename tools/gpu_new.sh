cd $GRAFT_REPO_ROOT; mkdir -p gpurun_out
timeout 1500 python -m pytest tests/test_bench_configs_gpu.py tests/test_dropin_gpu.py -x -q --timeout 1200 -rf --durations=8 > gpurun_out/pytest_new.txt 2>&1; echo rc=$?
tail -15 gpurun_out/pytest_new.txt
