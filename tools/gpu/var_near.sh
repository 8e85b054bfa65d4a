# near-pair A/B: general fused (config 2 at 1/h = 64 and 32), separate schedule near kernel, node path 1/h = 64
mkdir -p gpurun_out
summ() { python -c "import json,sys;d=json.loads(open(sys.argv[1]).read().strip().splitlines()[-1]);r=d['roofline'];p=d['parity'];print(sys.argv[2], '%.4g pairs/s  %.3f ms/step  frac %.4f kernel %.3f ms  near %.3f ms  par %.1e %.1e' % (d['value'], d['ms_per_step'], r['frac'], r['kernel_ms'], d.get('near_kernel',{}).get('ms',0), p['u_max_rel'], p['v_max_rel']))" "$@"; }
for args in "--config 2 --inv-h 64 --steps 20" "--config 2 --inv-h 32 --steps 40" "--config 2 --inv-h 64 --steps 20 --schedule separate" "--inv-h 64 --steps 20 --path nodes"; do
  echo "== $args"
  for rep in 1 2; do
  timeout 600 python bench.py $args --no-e2e --no-cpu-baseline > gpurun_out/vnear_def.json 2>&1 && summ gpurun_out/vnear_def.json "default" || tail -3 gpurun_out/vnear_def.json
  for lib in build/variants/*.so; do
    n=$(basename $lib .so)
    STOKES_ER_LIB=$PWD/$lib timeout 600 python bench.py $args --no-e2e --no-cpu-baseline > gpurun_out/vnear_$n.json 2>&1 && summ gpurun_out/vnear_$n.json "$n" || tail -3 gpurun_out/vnear_$n.json
  done
  done
done
timeout 900 python -m pytest tests/test_gpu_parity.py -q -x -k "config1 or per_delta or near_pair or wide_rho or degenerate or randomized or onsurface" > gpurun_out/pytest_near.log 2>&1; echo "pytest rc=$?"; tail -2 gpurun_out/pytest_near.log
