# final validation of the committed build: GPU suite, smoke, default bench line
D=gpurun_out/r01i; mkdir -p $D
timeout 1200 python -m pytest tests -m gpu -q --timeout 300 > $D/pytest_gpu.log 2>&1; tail -1 $D/pytest_gpu.log
timeout 120 python -c "import __graft_entry__ as g; g.smoke(); print('smoke ok')" > $D/smoke.log 2>&1; tail -1 $D/smoke.log
timeout 600 python bench.py --steps 10 --warmup 3 > $D/bench_default.json 2> $D/bench_default.err
python -c "
import json; d=json.loads(open('$D/bench_default.json').read().strip().splitlines()[-1])
print('default', '%.3e'%d['value'], round(d['roofline']['frac'],3), 'e2e %.3e'%d['e2e']['value'], d['clocks'])
for s in d['secondary']: print('  sec', '%.3e'%s['value'], round(s['roofline']['frac'],3))"
