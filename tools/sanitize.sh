cd $GRAFT_REPO_ROOT; mkdir -p gpurun_out
for tool in memcheck racecheck synccheck; do
  timeout 1200 /usr/local/cuda/bin/compute-sanitizer --tool $tool --print-limit 10 python tools/sanitize_kernels.py > gpurun_out/san_$tool.log 2>&1
  echo "$tool rc=$?"; grep -E "ERROR SUMMARY|sanitize run ok|Hazard|Error" gpurun_out/san_$tool.log | head -5
done
