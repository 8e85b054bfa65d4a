# near-queue prefetch A/B (SER_NEAR_PF, SER_NEAR_MINB): separate-schedule near kernel at config 2 1/h = 64,
# the fused default at config 2 1/h = 32 / 64, the node path at 1/h = 128 (nbr_kernel share)
mkdir -p gpurun_out
summ() { python -c "import json,sys;d=json.loads(open(sys.argv[1]).read().strip().splitlines()[-1]);r=d['roofline'];p=d['parity'];print(sys.argv[2], '%.4g pairs/s  %.3f ms/step  frac %.4f kernel %.3f ms  near %.3f ms  par %.1e %.1e' % (d['value'], d['ms_per_step'], r['frac'], r['kernel_ms'], d.get('near_kernel',{}).get('ms',0), p['u_max_rel'], p['v_max_rel']))" "$@"; }
for args in ${ARGSLIST:-"--config 2 --inv-h 64 --steps 20 --schedule separate" "--config 2 --inv-h 32 --steps 40" "--config 2 --inv-h 64 --steps 20" "--inv-h 128 --steps 10 --path nodes"}; do
  echo "== $args"
  timeout 600 python bench.py $args --no-e2e --no-cpu-baseline > gpurun_out/vnear_def.json 2>&1 && summ gpurun_out/vnear_def.json "default" || tail -3 gpurun_out/vnear_def.json
  for lib in build/variants/*.so; do
    n=$(basename $lib .so)
    STOKES_ER_LIB=$PWD/$lib timeout 600 python bench.py $args --no-e2e --no-cpu-baseline > gpurun_out/vnear_$n.json 2>&1 && summ gpurun_out/vnear_$n.json "$n" || tail -3 gpurun_out/vnear_$n.json
  done
done
