# ncu --set full of one kernel (regex $NCU) over tools/profile_sweep.py; summary + per-line source table
cd $GRAFT_REPO_ROOT; mkdir -p gpurun_out
TAG=${TAG:-x}
timeout 900 ncu --set full --clock-control none --import-source on -k regex:"$NCU" -s ${SKIP:-1} -c ${CNT:-1} -o gpurun_out/prof_$TAG python tools/profile_sweep.py > gpurun_out/ncu_$TAG.txt 2>&1
tail -1 gpurun_out/ncu_$TAG.txt
