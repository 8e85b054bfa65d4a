mkdir -p gpurun_out
summ() { python -c "import json,sys;d=json.load(open(sys.argv[1]));r=d['roofline'];print(sys.argv[2], '%.4g pairs/s  %.3f ms/step  kernel %.3f ms' % (d['value'], d['ms_per_step'], r['kernel_ms']))" "$@"; }
timeout 600 python -m pytest tests -m gpu -x -q 2>&1 | tail -2
for sch in fused separate; do
  timeout 300 python bench.py --steps 20 --no-e2e --no-cpu-baseline --schedule $sch $BENCH_ARGS > gpurun_out/sc_$sch.json 2>&1 && summ gpurun_out/sc_$sch.json $sch
done
for lib in build/variants/*.so; do
  [ -f "$lib" ] || continue
  n=$(basename $lib .so)
  STOKES_ER_LIB=$PWD/$lib timeout 300 python bench.py --steps 20 --no-e2e --no-cpu-baseline $BENCH_ARGS > gpurun_out/sw_$n.json 2>&1 && summ gpurun_out/sw_$n.json $n
done
