# Parity tests + bench + ncu (source-level) of the warm k_sweep and the cold pool tiers + pool stats (one GPU).
cd $GRAFT_REPO_ROOT; mkdir -p gpurun_out
TAG=${TAG:-ps}
timeout 1200 python -m pytest ${TESTS:-tests/test_gpu_parity.py} -m gpu -x -q --timeout 900 -rf > gpurun_out/pytest_$TAG.txt 2>&1; echo pytest rc=$?
tail -3 gpurun_out/pytest_$TAG.txt
timeout 900 python bench.py --steps 20 --warmup 5 > gpurun_out/bench_$TAG.txt 2>&1; echo bench rc=$?
timeout 300 python tools/pool_stats.py > gpurun_out/stats_$TAG.txt 2>&1; cat gpurun_out/stats_$TAG.txt | tail -12
SWEEPS=1 WARM=3 timeout 600 ncu --set full --clock-control none --import-source on -k regex:"k_sweep" -s 2 -c 1 -o gpurun_out/prof_sweep_$TAG python tools/profile_sweep.py > gpurun_out/ncu_sweep_$TAG.txt 2>&1; echo ncu rc=$?
SWEEPS=3 timeout 600 ncu --set full --clock-control none --import-source on -k regex:"k_pool_tile|k_pool_warp|k_pool_prep|k_mark|k_sample" -s 12 -c 6 -o gpurun_out/prof_cold_$TAG python tools/profile_sweep.py > gpurun_out/ncu_cold_$TAG.txt 2>&1; echo ncu rc=$?
