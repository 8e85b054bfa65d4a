# the bench lines of DESIGN.md Sec. 7 at the current code (TAG names the files)
mkdir -p gpurun_out
TAG=${TAG:-cur}
timeout 600 python bench.py --schedule separate --no-e2e --no-cpu-baseline > gpurun_out/bench_${TAG}_separate.json 2>/dev/null; echo "separate rc=$?"
timeout 900 python bench.py --config 3 --inv-h 128 --steps 10 > gpurun_out/bench_${TAG}_cfg3_h128.json 2>/dev/null; echo "cfg3 rc=$?"
timeout 900 python bench.py --config 5 --inv-h 128 --steps 10 > gpurun_out/bench_${TAG}_cfg5_h128.json 2>/dev/null; echo "cfg5 h128 rc=$?"
timeout 1200 python bench.py --config 5 --inv-h 256 --steps 4 --warmup 3 > gpurun_out/bench_${TAG}_cfg5_h256.json 2>/dev/null; echo "cfg5 h256 rc=$?"
timeout 900 python bench.py --config 6 --inv-h 128 --steps 5 --no-e2e --no-cpu-baseline > gpurun_out/bench_${TAG}_purefar_h128.json 2>/dev/null; echo "purefar rc=$?"
for f in gpurun_out/bench_${TAG}_*.json; do python -c "
import json,sys;d=json.loads(open(sys.argv[1]).read().strip().splitlines()[-1]);r=d['roofline'];e=d.get('e2e') or {};c=d.get('cpu_baseline') or {}
print(sys.argv[1].split('/')[-1], '%.4g pairs/s %.2f ms frac %.3f/%.3f e2e %s cpu %s' % (d['value'], d['ms_per_step'], r['frac'], r['frac_issued_convention'], '%.3g'%e['value'] if e else None, '%.3g'%c['value'] if c else None))" $f; done
