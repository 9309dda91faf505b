# compute-sanitizer over the key-first build kernels (one GPU).
cd $GRAFT_REPO_ROOT; mkdir -p gpurun_out
for tool in memcheck racecheck synccheck initcheck; do
  timeout 900 compute-sanitizer --tool $tool --error-exitcode 9 python tools/san_kf.py > gpurun_out/san_kf_$tool.txt 2>&1
  echo "$tool rc=$? $(grep -c 'ERROR SUMMARY: 0' gpurun_out/san_kf_$tool.txt) $(tail -1 gpurun_out/san_kf_$tool.txt)"
done
