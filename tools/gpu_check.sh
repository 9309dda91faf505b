cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
nvidia-smi -L > gpurun_out/gpu.txt 2>&1
timeout 1200 python -m pytest tests -m gpu -q --timeout 600 -rf > gpurun_out/pytest_gpu.txt 2>&1
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke.txt 2>&1
timeout 600 python bench.py --steps 5 --warmup 3 > gpurun_out/bench.txt 2>&1
tail -5 gpurun_out/pytest_gpu.txt; tail -3 gpurun_out/smoke.txt; tail -3 gpurun_out/bench.txt
