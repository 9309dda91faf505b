# Full GPU tests + C3 + C4 (trace) + bench line (one GPU).
cd $GRAFT_REPO_ROOT; mkdir -p gpurun_out
TAG=${TAG:-rd}
timeout 2000 python -m pytest tests -m gpu -x -q --timeout 1200 -rf --durations=5 > gpurun_out/pytest_$TAG.txt 2>&1; echo pytest rc=$?
tail -8 gpurun_out/pytest_$TAG.txt
EMU_BUILD_TRACE=1 timeout 600 python bench_configs.py c4 --steps 5 > gpurun_out/c4_$TAG.txt 2>&1; echo c4 rc=$?
grep "emu build" gpurun_out/c4_$TAG.txt | tail -11; tail -1 gpurun_out/c4_$TAG.txt | cut -c1-700
timeout 900 python bench_configs.py c3 --steps 4 > gpurun_out/c3_$TAG.txt 2>&1; echo c3 rc=$?
tail -1 gpurun_out/c3_$TAG.txt | cut -c1-900
if [ -n "$BENCH" ]; then timeout 900 python bench.py --steps 20 --warmup 5 > gpurun_out/bench_$TAG.txt 2>&1; echo bench rc=$?; tail -1 gpurun_out/bench_$TAG.txt | cut -c1-400; fi
