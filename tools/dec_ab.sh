cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
timeout 600 python -m pytest tests -m gpu -q -x -k "codec or decode" > gpurun_out/ab_pytest.log 2>&1; echo "pytest rc=$?" >> gpurun_out/ab_pytest.log
tail -2 gpurun_out/ab_pytest.log
for v in 3 2; do
  sed -i "s/__launch_bounds__(kD128Threads, [0-9])/__launch_bounds__(kD128Threads, $v)/" paper_2605_21226_b200/csrc/decode.cu
  make -j16 > /dev/null 2>&1
  timeout 300 python bench.py --no-cpu-baseline --steps 5 > gpurun_out/ab_$v.log 2>&1
  python -c "
import json
l=[x for x in open('gpurun_out/ab_$v.log') if x.startswith('{')]
d=json.loads(l[-1]); c=d['compress']
print('minB $v decode us', round(c['decode']['ms']*1e3,1), 'GB/s', round(c['decode']['gbs']), 'compress us', round(c['ms']*1e3,1))
"
done
OQ_DECODE_GENERIC=1 timeout 300 python bench.py --no-cpu-baseline --steps 5 2>&1 | grep '^{' | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('generic decode us', round(d['compress']['decode']['ms']*1e3,1))"
