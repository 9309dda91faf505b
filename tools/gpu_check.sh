cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
timeout 1500 python -m pytest tests -m gpu -q --timeout 600 -rf -x > gpurun_out/pytest_gpu.txt 2>&1
timeout 600 python bench.py --steps 5 --warmup 3 > gpurun_out/bench.txt 2>&1
timeout 300 python tools/pool_stats.py > gpurun_out/stats.txt 2>&1
tail -15 gpurun_out/pytest_gpu.txt; tail -3 gpurun_out/bench.txt | cut -c1-900; cat gpurun_out/stats.txt
