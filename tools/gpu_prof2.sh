cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
timeout 900 ncu --set full --clock-control none --import-source on -k regex:"k_sample|k_mark" -s 2 -c 2 -o gpurun_out/prof_r5 python tools/profile_sweep.py > gpurun_out/ncu_full.txt 2>&1
tail -2 gpurun_out/ncu_full.txt
