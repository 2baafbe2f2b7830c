for w in qft rzz qaoa diag; do tail -1 gpurun_out/bench_$w.log | python -c "
import json,sys
try:
  d=json.loads(sys.stdin.read()); print('$w', round(d['ms_per_step'],3), {k:round(v['ms']/d['steps'],3) for k,v in d['kernels'].items()}, round(d['roofline']['frac'],3))
except Exception as e: print('$w ERR', e)"; done
