# far-item size sweep (the grid tail vs per-item overhead), both schedules
mkdir -p gpurun_out
summ() { python -c "import json,sys;d=json.loads(open(sys.argv[1]).read().strip().splitlines()[-1]);r=d['roofline'];c=d['config'];print(sys.argv[2], '%.4g pairs/s  %.3f ms/step  kernel %.3f ms  frac %.4f  items %s chunk %s' % (d['value'], d['ms_per_step'], r['kernel_ms'], r['frac'], c.get('work_items'), c.get('chunk_tiles')))" "$@"; }
for cfg in "--config 2 --inv-h 64" "--config 6 --inv-h 128"; do
  for sch in fused separate; do
    for ct in 0 8 12 16 32 46; do
      a="$cfg --schedule $sch"; [ $ct -gt 0 ] && a="$a --chunk-tiles $ct"
      timeout 300 python bench.py $a --steps 10 --no-e2e --no-cpu-baseline > gpurun_out/cs.json 2>&1 && summ gpurun_out/cs.json "$a"
    done
  done
done
