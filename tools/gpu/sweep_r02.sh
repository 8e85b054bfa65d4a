# config 5 sweep (auto path: general below 1.5e5 nodes, node path above) + configs 2/3/4 lines on the final build
mkdir -p gpurun_out/lines
summ() { python -c "import json,sys;d=json.loads(open(sys.argv[1]).read().strip().splitlines()[-1]);r=d['roofline'];c=d.get('cpu_baseline') or {};print(sys.argv[1], '%.4g pairs/s  %.3f ms  frac %.3f  path %s  e2e %.4g  oracle %s  par %s' % (d['value'], d['ms_per_step'], r['frac'], d['config'].get('path'), (d.get('e2e') or {}).get('value', 0), c.get('value'), (d.get('parity') or {}).get('u_max_rel')))" "$@"; }
for a in "--config 5 --inv-h 32 --steps 40" "--config 5 --inv-h 64 --steps 20" "--config 5 --inv-h 64 --steps 20 --path nodes" "--config 5 --inv-h 128 --steps 10" "--config 5 --inv-h 128 --steps 10 --path general" "--config 2 --inv-h 64 --steps 20" "--config 3 --inv-h 64 --steps 20" "--config 3 --inv-h 128 --steps 5" "--config 4 --inv-h 64 --eps 0.05 --steps 10"; do
  n=$(echo $a | tr -d ' -' | tr '.' 'p')
  timeout 900 python bench.py $a > gpurun_out/lines/$n.json 2> gpurun_out/lines/$n.err && summ gpurun_out/lines/$n.json || tail -3 gpurun_out/lines/$n.err
done
