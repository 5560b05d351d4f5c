#!/bin/bash
cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
OQ_ATTN_IMPL=regs timeout 900 /usr/local/cuda/bin/ncu --set full --import-source on --clock-control none -k regex:attn_partials -s 4 -c 1 -o gpurun_out/prof_attn_regs -f python bench.py --steps 3 --warmup 3 --no-cpu-baseline --no-compress > gpurun_out/ncu_attn_regs.log 2>&1
echo "rc=$?"; tail -2 gpurun_out/ncu_attn_regs.log
