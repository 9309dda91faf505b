cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
timeout 600 python -m pytest tests/test_gpu_parity.py -q --timeout 300 -k small_arena > gpurun_out/pytest_small.txt 2>&1
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches_r1.csv python bench.py --steps 2 --warmup 1 --no-extras > gpurun_out/ncu_bench.txt 2>&1
timeout 900 ncu --set full --clock-control none --import-source on -k regex:"k_pool_warp|k_sample|k_mark" -s 3 -c 3 -o gpurun_out/prof_r1 python tools/profile_sweep.py > gpurun_out/ncu_full.txt 2>&1
tail -3 gpurun_out/pytest_small.txt; tail -3 gpurun_out/ncu_full.txt; ls -la gpurun_out
