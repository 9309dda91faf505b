cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
timeout 900 ncu --set full --clock-control none --import-source on -k regex:"k_pool_warp" -s 1 -c 1 -o gpurun_out/prof_r4 python tools/profile_sweep.py > gpurun_out/ncu_full.txt 2>&1
tail -3 gpurun_out/ncu_full.txt
