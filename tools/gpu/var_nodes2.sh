# node path A/B at 1/h = 64, 128 (+256): default vs build/variants/*.so
mkdir -p gpurun_out
summ() { python -c "import json,sys;d=json.loads(open(sys.argv[1]).read().strip().splitlines()[-1]);r=d['roofline'];p=d['parity'];print(sys.argv[2], '%.4g pairs/s  %.3f ms/step  frac %.4f kernel %.2f ms  nbr %.2f ms  par %.1e %.1e' % (d['value'], d['ms_per_step'], r['frac'], r['kernel_ms'], d.get('near_kernel',{}).get('ms',0), p['u_max_rel'], p['v_max_rel']))" "$@"; }
for args in "--inv-h 64 --steps 20 --path nodes" "--inv-h 128 --steps 10" ${EXTRA:+"$EXTRA"}; do
  echo "== $args"
  for rep in 1 2; do
  timeout 600 python bench.py $args --no-e2e --no-cpu-baseline > gpurun_out/vn2_def.json 2>&1 && summ gpurun_out/vn2_def.json "default" || tail -3 gpurun_out/vn2_def.json
  for lib in build/variants/*.so; do
    n=$(basename $lib .so)
    STOKES_ER_LIB=$PWD/$lib timeout 600 python bench.py $args --no-e2e --no-cpu-baseline > gpurun_out/vn2_$n.json 2>&1 && summ gpurun_out/vn2_$n.json "$n" || tail -3 gpurun_out/vn2_$n.json
  done
  done
done
