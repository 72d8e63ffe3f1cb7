timeout 1200 python bench.py > gpurun_out/r2cc_bench.log 2>&1; tail -c 3000 gpurun_out/r2cc_bench.log | tail -1 | python -c "
import json,sys
d=json.loads(sys.stdin.read())
print('value',d['value']/1e9,'frac',d['roofline']['frac'],'traffic',d['roofline'].get('traffic'))
print('cgi',d['cg_iteration_c5']['ms_per_iteration'])
print('cg',d['cg']['ms_per_iteration'],d['cg']['iterations'],d['cg']['solve_ms'])
print('c4',d['c4_step']['ms_per_step_steady'])
print('configs',{k:round(v['ms'],4) for k,v in d['configs'].items()})
print('e2e',d['e2e']['value']/1e9)
print('cpu',d['cpu_baseline'])
"
