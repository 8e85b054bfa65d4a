mkdir -p gpurun_out
summ() { python -c "import json,sys;d=json.load(open(sys.argv[1]));r=d['roofline'];print(sys.argv[2], '%.4g pairs/s  %.3f ms/step  kernel %.3f ms' % (d['value'], d['ms_per_step'], r['kernel_ms']))" "$@"; }
for ph in 0 16 32; do
  timeout 300 python bench.py --steps 20 --no-e2e --no-cpu-baseline --near-phases $ph > gpurun_out/sw_ph$ph.json 2>&1 && summ gpurun_out/sw_ph$ph.json default_ph$ph
  for lib in build/variants/*.so; do
    n=$(basename $lib .so)
    STOKES_ER_LIB=$PWD/$lib timeout 300 python bench.py --steps 20 --no-e2e --no-cpu-baseline --near-phases $ph > gpurun_out/sw_$n.json 2>&1 && summ gpurun_out/sw_$n.json ${n}_ph$ph
  done
done
timeout 300 python bench.py --steps 20 --no-e2e --no-cpu-baseline --schedule separate > gpurun_out/sw_sep.json 2>&1 && summ gpurun_out/sw_sep.json separate
