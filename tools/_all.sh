for c in cfg1 cfg2 cfg4 cfg5; do s=$(date +%s); python bench.py --config $c > gpurun_out/head_$c.json 2> gpurun_out/head_$c.err; echo "$c rc=$? wall $(( $(date +%s) - s )) s"; tail -c 300 gpurun_out/head_$c.err; python - <<P
import json
try:
    d=json.loads(open("gpurun_out/head_$c.json").read().strip().splitlines()[-1])
    print(d['value'], d['unit'], 'e2e', d['e2e']['value'], 'frac', d['roofline']['frac'], 'conv', d.get('converged'), d.get('clocks'))
except Exception as e: print('parse', e)
P
done
