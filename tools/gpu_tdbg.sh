cd $GRAFT_REPO_ROOT; mkdir -p gpurun_out
EMU_LIB_PATH=$PWD/paper_2605_00616_b200/libemu_b200_check.so EMU_STEP_SERVER=0 timeout 600 python tools/tile_debug.py 2>&1 | grep -v "^ " | sort | uniq -c | sort -rn | head -20
EMU_TILE_STATS=1 EMU_STEP_SERVER=0 timeout 600 python tools/tile_debug.py 2>&1 | tail -8
