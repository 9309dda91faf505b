# Parity tests + C3 timing (one GPU).
cd $GRAFT_REPO_ROOT; mkdir -p gpurun_out
TAG=${TAG:-c3t}
timeout 1500 python -m pytest ${TESTS:-tests/test_gpu_parity.py tests/test_bench_configs_gpu.py tests/test_reference_suite_gpu.py} -m gpu -x -q --timeout 1200 -rf > gpurun_out/pytest_$TAG.txt 2>&1; echo pytest rc=$?
tail -3 gpurun_out/pytest_$TAG.txt
EMU_TILE_STATS=1 timeout 900 python bench_configs.py c3 --steps 4 > gpurun_out/c3_$TAG.txt 2>&1; echo c3 rc=$?
grep "new keys" gpurun_out/c3_$TAG.txt | sort | uniq -c | head -4; tail -1 gpurun_out/c3_$TAG.txt
SWEEPS=10 timeout 300 python tools/kernel_times.py 2>&1 | tail -1
WORK=sparse FLOOR=256 timeout 600 python tools/pool_stats.py 2>&1 | tail -10
