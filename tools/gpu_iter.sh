# One build->measure iteration: GPU tests, stats, bench (one GPU).
cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
TAG=${TAG:-it}
timeout 1200 python -m pytest tests -m gpu -x -q --timeout 900 -rf --durations=6 > gpurun_out/pytest_$TAG.txt 2>&1
tail -12 gpurun_out/pytest_$TAG.txt
timeout 300 python tools/pool_stats.py > gpurun_out/stats_$TAG.txt 2>&1; cat gpurun_out/stats_$TAG.txt
timeout 600 python bench.py --steps 10 --warmup 3 > gpurun_out/bench_$TAG.txt 2>&1
tail -1 gpurun_out/bench_$TAG.txt | python -c "import json,sys; d=json.loads(sys.stdin.read()); print(d['ms_per_step'], d['value']/1e9, d['roofline']['kernels_ms'], d['e2e']['value']/1e9, d['e2e']['ms_per_step'], d.get('p50_us_per_step_query'))"
if [ -n "$NCU" ]; then
  timeout 900 ncu --set full --clock-control none --import-source on -k regex:"$NCU" -s 2 -c 2 -o gpurun_out/prof_$TAG python tools/profile_sweep.py > gpurun_out/ncu_$TAG.txt 2>&1
  tail -1 gpurun_out/ncu_$TAG.txt
fi
