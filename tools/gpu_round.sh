#!/bin/bash
# One gpurun call: smoke (+memcheck), GPU parity tests, bench, ncu captures.
# Stages selectable with STAGES="smoke memcheck pytest bench ncu" (default all).
cd "$(dirname "$0")/.."
mkdir -p gpurun_out
STAGES=${STAGES:-"smoke memcheck pytest bench ncu"}
nvidia-smi > gpurun_out/nvidia-smi.txt 2>&1
nproc > gpurun_out/host.txt; lscpu | grep -E "Model name|^CPU\(s\)" >> gpurun_out/host.txt
for s in $STAGES; do case $s in
smoke) timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke.log 2>&1; echo "smoke rc=$?" >> gpurun_out/smoke.log;;
memcheck) timeout 600 /usr/local/cuda/bin/compute-sanitizer --tool memcheck --print-limit 20 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/memcheck.log 2>&1; echo "memcheck rc=$?" >> gpurun_out/memcheck.log;;
pytest) timeout 1200 python -m pytest tests -m gpu -q ${PYTEST_ARGS} > gpurun_out/pytest_gpu.log 2>&1; echo "pytest rc=$?" >> gpurun_out/pytest_gpu.log;;
bench) timeout 600 python bench.py ${BENCH_ARGS} > gpurun_out/bench.log 2>&1; echo "bench rc=$?" >> gpurun_out/bench.log;;
ncuattn)
  timeout 900 /usr/local/cuda/bin/ncu --set full --clock-control none --import-source on -k regex:attn_partials -s 4 -c 1 -o gpurun_out/prof_attn -f python bench.py --steps 3 --warmup 3 --no-cpu-baseline --no-compress --no-other-configs > gpurun_out/ncu_attn.log 2>&1; echo "ncu attn rc=$?" >> gpurun_out/ncu_attn.log
  ;;
ncucodec)
  timeout 900 /usr/local/cuda/bin/ncu --set full --clock-control none --import-source on -k regex:"compress_kernel|decode_kernel" -s 2 -c 2 -o gpurun_out/prof_codec -f python tools/codec_kernels.py > gpurun_out/ncu_codec.log 2>&1; echo "ncu codec rc=$?" >> gpurun_out/ncu_codec.log
  ;;
ncu)
  timeout 600 /usr/local/cuda/bin/ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv --log-file gpurun_out/launches.csv python bench.py --steps 3 --warmup 3 --no-cpu-baseline --no-other-configs > gpurun_out/ncu_launch.log 2>&1; echo "ncu launches rc=$?" >> gpurun_out/ncu_launch.log
  for cfg in c3 c4 c5; do
    timeout 900 /usr/local/cuda/bin/ncu --set full --clock-control none --import-source on -k regex:attn_partials -s 4 -c 1 -o gpurun_out/prof_attn_$cfg -f python bench.py --config $cfg --steps 3 --warmup 3 --no-cpu-baseline --no-compress --no-other-configs > gpurun_out/ncu_attn_$cfg.log 2>&1; echo "ncu attn $cfg rc=$?" >> gpurun_out/ncu_attn_$cfg.log
  done
  timeout 900 /usr/local/cuda/bin/ncu --set full --clock-control none --import-source on -k regex:"compress_fast_kernel|compress_fixup_kernel|decode128_kernel" -s 3 -c 3 -o gpurun_out/prof_codec -f python tools/codec_kernels.py 3 > gpurun_out/ncu_codec.log 2>&1; echo "ncu codec rc=$?" >> gpurun_out/ncu_codec.log
  ;;
esac; done
for f in gpurun_out/*.log; do echo "== $f"; tail -4 $f; done
