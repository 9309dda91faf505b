# GPU test suite + 1-GPU bench line (one B200).
cd $GRAFT_REPO_ROOT; mkdir -p gpurun_out
TAG=${TAG:-full}
timeout 1800 python -m pytest tests -m gpu -x -q --timeout 1200 -rf --durations=8 > gpurun_out/pytest_$TAG.txt 2>&1; echo pytest rc=$?
tail -15 gpurun_out/pytest_$TAG.txt
timeout 900 python bench.py --steps 20 --warmup 5 > gpurun_out/bench_$TAG.txt 2>&1; echo bench rc=$?
tail -1 gpurun_out/bench_$TAG.txt
