# Out-of-grid pool parity repro on one GPU (tools/oog_strict.py): check build, plain build, synccheck.
cd $GRAFT_REPO_ROOT; mkdir -p gpurun_out
export EMU_STEP_SERVER=0
for GEN in llama sparse; do
timeout 900 env GEN=$GEN EMU_LIB_PATH=$PWD/paper_2605_00616_b200/libemu_b200_check.so ROUNDS=${ROUNDS:-10} python tools/oog_strict.py > gpurun_out/oog_check_$GEN.txt 2>&1; echo check $GEN rc=$?
tail -4 gpurun_out/oog_check_$GEN.txt
timeout 900 env GEN=$GEN ROUNDS=${ROUNDS2:-30} python tools/oog_strict.py > gpurun_out/oog_plain_$GEN.txt 2>&1; echo plain $GEN rc=$?
tail -3 gpurun_out/oog_plain_$GEN.txt
done
timeout 900 compute-sanitizer --tool synccheck --print-limit 20 env ROUNDS=2 QS=20000 python tools/oog_strict.py > gpurun_out/oog_sync.txt 2>&1; echo sync rc=$?
tail -4 gpurun_out/oog_sync.txt
timeout 900 compute-sanitizer --tool racecheck --print-limit 20 env ROUNDS=1 QS=20000 python tools/oog_strict.py > gpurun_out/oog_race.txt 2>&1; echo race rc=$?
tail -4 gpurun_out/oog_race.txt
