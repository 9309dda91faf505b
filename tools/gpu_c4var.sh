# C4 build time for each variants/<name>/libemu_b200.so and the default build (one GPU).
cd $GRAFT_REPO_ROOT; mkdir -p gpurun_out
for d in $(ls -d variants/*/ 2>/dev/null) ""; do
  n=$(basename "${d:-default}")
  lib=${d:+$PWD/$d/libemu_b200.so}
  EMU_LIB_PATH=$lib timeout 300 python bench_configs.py c4 --steps 5 2>/dev/null | tail -1 | python -c "
import json,sys; d=json.loads(sys.stdin.read()); print('$n', d['ms_per_build'], d['ms_per_build_all'], {k: v for k, v in d['kernels_ms'].items() if v[0] > 0.2})"
done
