# Parity tests (subset) + C2 kernel times + bench line (one GPU).
cd $GRAFT_REPO_ROOT; mkdir -p gpurun_out
TAG=${TAG:-kt}
timeout 1500 python -m pytest ${TESTS:-tests/test_gpu_parity.py tests/test_bench_configs_gpu.py tests/test_reference_suite_gpu.py} -m gpu -x -q --timeout 1200 -rf > gpurun_out/pytest_$TAG.txt 2>&1; echo pytest rc=$?
tail -3 gpurun_out/pytest_$TAG.txt
SWEEPS=10 timeout 300 python tools/kernel_times.py 2>&1 | tail -1
EMU_TILE_STATS=1 SWEEPS=1 timeout 300 python tools/kernel_times.py 2>&1 | grep "new keys" | tail -1
if [ -n "$BENCH" ]; then timeout 900 python bench.py --steps 20 --warmup 5 > gpurun_out/bench_$TAG.txt 2>&1; echo bench rc=$?; tail -1 gpurun_out/bench_$TAG.txt | cut -c1-300; fi
