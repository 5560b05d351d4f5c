cd $GRAFT_REPO_ROOT; mkdir -p gpurun_out
timeout 900 python -m pytest tests -m gpu -q -x -k "codec" 2>&1 | tail -2
timeout 600 python tools/compress_diag.py 2>&1 | tee gpurun_out/cdiag.log
timeout 600 /usr/local/cuda/bin/ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/cdiag_launches.csv python tools/codec_kernels.py 3 > /dev/null 2>&1
python tools/ncu_summary.py launches gpurun_out/cdiag_launches.csv | grep oqd
