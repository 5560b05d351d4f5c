cd $GRAFT_REPO_ROOT; mkdir -p gpurun_out
timeout 900 /usr/local/cuda/bin/ncu --set full --clock-control none --import-source on -k regex:"compress_fast_kernel" -s 1 -c 1 -o gpurun_out/prof_cfast -f python tools/codec_kernels.py 3 > gpurun_out/ncu_cfast.log 2>&1; echo "rc=$?"; tail -2 gpurun_out/ncu_cfast.log
