python -m pytest tests -m gpu -x -q > gpurun_out/pytest_gpu.log 2>&1; tail -3 gpurun_out/pytest_gpu.log
python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke.log 2>&1; tail -2 gpurun_out/smoke.log
python bench.py > gpurun_out/bench_default.json 2> gpurun_out/bench_default.err; tail -c 300 gpurun_out/bench_default.err
python - <<P
import json
d=json.loads(open("gpurun_out/bench_default.json").read().strip().splitlines()[-1])
print(d['value'], d['step_ms'], 'e2e', d['e2e']['value'], 'setup', d['setup_s'], 'frac', d['roofline']['frac'])
P
RMG_SETUP_LOG=1 python bench.py --config cfg5 --no-cpu-baseline > gpurun_out/cfg5_defer.json 2> gpurun_out/cfg5_defer.err; grep "rmg setup" gpurun_out/cfg5_defer.err | grep -v upload
python - <<P
import json
d=json.loads(open("gpurun_out/cfg5_defer.json").read().strip().splitlines()[-1])
print(d['value'], 'e2e', d['e2e']['value'], 'setup', d['setup_s'], 'frac', d['roofline']['frac'], d.get('iterations'))
P
