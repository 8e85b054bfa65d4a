# DESIGN 8.0a bench lines on the current build (profiles/r02/lines/<args>.json)
mkdir -p gpurun_out/lines
run() { n=$(echo "$*" | tr -d ' -' | tr '.' 'p'); timeout 900 python bench.py "$@" > gpurun_out/lines/$n.json 2> gpurun_out/lines/$n.err; echo "$n rc=$?"; }
run --config 5 --inv-h 32 --steps 40
run --config 5 --inv-h 64 --steps 20
run --config 5 --inv-h 64 --steps 20 --path nodes
run --config 5 --inv-h 128 --steps 10
run --config 5 --inv-h 128 --steps 10 --path general
run --config 5 --inv-h 256 --steps 4
run --config 5 --inv-h 256 --steps 4 --path general --no-cpu-baseline
run --config 2 --inv-h 64 --steps 20
run --config 3 --inv-h 64 --steps 20
run --config 3 --inv-h 128 --steps 5
run --config 4 --inv-h 64 --eps 0.05 --steps 10
for f in gpurun_out/lines/*.json; do python -c "
import json,sys;d=json.loads(open(sys.argv[1]).read().strip().splitlines()[-1]);r=d['roofline'];e=d.get('e2e') or {};c=d.get('cpu_baseline') or {}
print(sys.argv[1].split('/')[-1], d['config'].get('path'), '%.4g pairs/s %.2f ms frac %.3f e2e %s cpu %s clk %s par %.1e' % (d['value'], d['ms_per_step'], r['frac'], '%.3g'%e['value'] if e else None, '%.3g'%c['value'] if c else None, d['clocks']['sm_mhz'], max(d['parity']['u_max_rel'], d['parity']['v_max_rel'])))" $f; done
