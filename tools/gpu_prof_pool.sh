# Pool-build profile: per-phase stats (EMU_STATS build) + ncu full capture of k_pool_warp.
cd $GRAFT_REPO_ROOT; mkdir -p gpurun_out
TAG=${TAG:-pw}
timeout 300 python tools/pool_stats.py > gpurun_out/stats_$TAG.txt 2>&1; cat gpurun_out/stats_$TAG.txt
timeout 300 env WORK=sparse python tools/pool_stats.py > gpurun_out/stats_sparse_$TAG.txt 2>&1; cat gpurun_out/stats_sparse_$TAG.txt
timeout 900 ncu --set full --clock-control none --import-source on -k regex:"${NCU:-k_pool_warp|k_sample|k_mark|k_pool_prep}" -s 4 -c 4 -o gpurun_out/prof_$TAG python tools/profile_sweep.py > gpurun_out/ncu_$TAG.txt 2>&1
tail -2 gpurun_out/ncu_$TAG.txt
