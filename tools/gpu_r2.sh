# Round-2 measurement pass: GPU tests, bench line, launch list, ncu --set full of the sweep kernels (one GPU).
cd $GRAFT_REPO_ROOT; mkdir -p gpurun_out
TAG=${TAG:-r2}
if [ -z "$SKIP_TESTS" ]; then
timeout 1800 python -m pytest tests -m gpu -x -q --timeout 1200 -rf --durations=8 > gpurun_out/pytest_$TAG.txt 2>&1; echo pytest rc=$?
tail -6 gpurun_out/pytest_$TAG.txt
fi
timeout 900 python bench.py --steps 20 --warmup 5 > gpurun_out/bench_$TAG.txt 2>&1; echo bench rc=$?
tail -1 gpurun_out/bench_$TAG.txt | cut -c1-600
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv --log-file gpurun_out/launches_$TAG.csv python bench.py --steps 2 --warmup 1 --no-extras > gpurun_out/launches_bench_$TAG.log 2>&1; echo launches rc=$?
timeout 900 ncu --set full --clock-control none --import-source on -k regex:"${NCU:-k_pool|k_sample|k_mark|k_sweep}" -s ${NCU_SKIP:-6} -c ${NCU_COUNT:-6} -o gpurun_out/prof_$TAG python tools/profile_sweep.py > gpurun_out/ncu_full_$TAG.txt 2>&1; echo ncu rc=$?
tail -2 gpurun_out/ncu_full_$TAG.txt
