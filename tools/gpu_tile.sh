# Tile-tier iteration: tier stats, parity tests, bench line.
cd $GRAFT_REPO_ROOT; mkdir -p gpurun_out
TAG=${TAG:-tile}
timeout 300 python tools/pool_stats.py 2>&1 | tail -12
timeout 300 env WORK=sparse python tools/pool_stats.py 2>&1 | tail -3
timeout 1500 python -m pytest tests -m gpu -x -q --timeout 1200 -rf > gpurun_out/pytest_$TAG.txt 2>&1; echo pytest rc=$?
tail -4 gpurun_out/pytest_$TAG.txt
timeout 600 python bench.py --steps 5 --warmup 3 > gpurun_out/bench_full_$TAG.txt 2>&1
tail -1 gpurun_out/bench_full_$TAG.txt | python -c "import json,sys; d=json.loads(sys.stdin.read()); print(d['ms_per_step'], d['roofline']['kernels_ms'], d['e2e']['value']/1e9)"
