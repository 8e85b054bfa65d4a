mkdir -p gpurun_out
summ() { python -c "import json,sys;d=json.loads(open(sys.argv[1]).read().strip().splitlines()[-1]);r=d['roofline'];print(sys.argv[2], '%.4g pairs/s  %.3f ms/step  frac %.4f issued %.4f' % (d['value'], d['ms_per_step'], r['frac'], r['frac_issued_convention']))" "$@"; }
for args in "--config 6 --inv-h 128" "--config 2 --inv-h 64"; do
  tag=$(echo $args | tr -d " -")
  timeout 300 python bench.py $args --steps 10 --no-e2e --no-cpu-baseline > gpurun_out/fv_def_$tag.json 2>&1 && summ gpurun_out/fv_def_$tag.json "default $args"
  for lib in build/variants/*.so; do
    n=$(basename $lib .so)
    STOKES_ER_LIB=$PWD/$lib timeout 300 python bench.py $args --steps 10 --no-e2e --no-cpu-baseline > gpurun_out/fv_${n}_$tag.json 2>&1 && summ gpurun_out/fv_${n}_$tag.json "$n $args"
  done
done
