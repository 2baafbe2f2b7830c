import glob, json, sys
for f in sorted(glob.glob(sys.argv[1] if len(sys.argv) > 1 else 'gpurun_out/ab_*.log')):
    try:
        d = json.loads(open(f).read().strip().splitlines()[-1])
        print(f, round(d['ms_per_step'], 3), {k: round(v['ms'] / d['steps'], 3) for k, v in d['kernels'].items() if v['ms'] > 1})
    except Exception as e:
        print(f, 'ERR', e)
