# C3 M=256 sweep time for each variants/<name>/libemu_b200.so and the default build (one GPU).
cd $GRAFT_REPO_ROOT
for d in variants/*/; do
  n=$(basename $d)
  TAG=$n EMU_LIB_PATH=$PWD/$d/libemu_b200.so SWEEPS=3 timeout 300 python tools/c3_sweep.py 2>&1 | tail -1
done
TAG=default SWEEPS=3 timeout 300 python tools/c3_sweep.py 2>&1 | tail -1
