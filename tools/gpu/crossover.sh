# node path vs general path on config 5 below the bench's auto switch (1.5e5 nodes)
mkdir -p gpurun_out
summ() { python -c "import json,sys;d=json.loads(open(sys.argv[1]).read().strip().splitlines()[-1]);print(sys.argv[2], '%.4g pairs/s  %.3f ms/step' % (d['value'], d['ms_per_step']))" "$@"; }
for H in 32 64 96; do
  for P in general nodes; do
    timeout 600 python bench.py --inv-h $H --path $P --steps 20 --no-e2e --no-cpu-baseline > gpurun_out/xo_${H}_$P.json 2>&1 && summ gpurun_out/xo_${H}_$P.json "1/h=$H $P" || tail -3 gpurun_out/xo_${H}_$P.json
  done
done
