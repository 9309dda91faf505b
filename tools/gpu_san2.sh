# Round-2 sanitizer pass over tools/san_paths.py (one GPU).
cd $GRAFT_REPO_ROOT; mkdir -p gpurun_out
export EMU_STEP_SERVER=0
for tool in memcheck racecheck synccheck initcheck; do
  timeout 1500 compute-sanitizer --tool $tool --error-exitcode 9 --print-limit 40 python tools/san_paths.py > gpurun_out/san2_$tool.txt 2>&1
  echo "$tool rc=$?"; grep -E "ERROR SUMMARY|ok|MISMATCH|Error" gpurun_out/san2_$tool.txt | tail -12
done
