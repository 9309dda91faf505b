cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
timeout 1500 python -m pytest tests -m gpu -q --timeout 900 -rf --durations=8 > gpurun_out/pytest_gpu.txt 2>&1
timeout 600 python bench.py --steps 5 --warmup 3 > gpurun_out/bench.txt 2>&1
tail -25 gpurun_out/pytest_gpu.txt; tail -3 gpurun_out/bench.txt | cut -c1-300
