# quick A/B of the default library against build/variants/*.so (config 2, default bench)
mkdir -p gpurun_out
summ() { python -c "import json,sys;d=json.loads(open(sys.argv[1]).read().strip().splitlines()[-1]);r=d['roofline'];print(sys.argv[2], '%.4g pairs/s  %.3f ms/step  frac %.4f issued %.4f' % (d['value'], d['ms_per_step'], r['frac'], r['frac_issued_convention']))" "$@"; }
args=${ARGS:-"--config 2 --inv-h 64"}
for rep in 1 2; do
  timeout 300 python bench.py $args --steps 20 --no-e2e --no-cpu-baseline > gpurun_out/vq_def.json 2>&1 && summ gpurun_out/vq_def.json "default"
  for lib in build/variants/*.so; do
    n=$(basename $lib .so)
    STOKES_ER_LIB=$PWD/$lib timeout 300 python bench.py $args --steps 20 --no-e2e --no-cpu-baseline > gpurun_out/vq_$n.json 2>&1 && summ gpurun_out/vq_$n.json "$n"
  done
done
