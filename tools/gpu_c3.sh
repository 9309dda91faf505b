# C3 (sparse long context) at M = 32 / 256: pool-build phase accounting + the bench_configs c3 line (one GPU).
cd $GRAFT_REPO_ROOT; mkdir -p gpurun_out
TAG=${TAG:-c3}
WORK=sparse FLOOR=256 timeout 600 python tools/pool_stats.py 2>&1 | tail -12
EMU_TILE_STATS=1 timeout 900 python bench_configs.py c3 --steps 4 > gpurun_out/c3_$TAG.txt 2>&1; echo c3 rc=$?
grep "new keys" gpurun_out/c3_$TAG.txt | sort | uniq -c | head; tail -1 gpurun_out/c3_$TAG.txt
if [ -n "$NCU" ]; then
Q=2000000 timeout 900 ncu --set full --clock-control none --import-source on -k regex:"k_pool_grp" -c 1 -o gpurun_out/prof_grp_$TAG python tools/c3_sweep.py > gpurun_out/ncu_grp_$TAG.txt 2>&1; echo ncu rc=$?
fi
