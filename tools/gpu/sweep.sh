# sweep tuning variants built by tools/build_variant.py: bench (fused) per variant
mkdir -p gpurun_out
summ() { python -c "import json,sys;d=json.load(open(sys.argv[1]));r=d['roofline'];print(sys.argv[2], '%.4g pairs/s  %.3f ms/step  kernel %.3f ms' % (d['value'], d['ms_per_step'], r['kernel_ms']))" "$@"; }
timeout 300 python bench.py --steps 20 --no-e2e --no-cpu-baseline > gpurun_out/sw_default.json 2>&1 && summ gpurun_out/sw_default.json default
for lib in build/variants/*.so; do
  n=$(basename $lib .so)
  STOKES_ER_LIB=$PWD/$lib timeout 300 python bench.py --steps 20 --no-e2e --no-cpu-baseline $SWEEP_ARGS > gpurun_out/sw_$n.json 2>&1 && summ gpurun_out/sw_$n.json $n
done
