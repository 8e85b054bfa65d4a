# general path: targets per thread (2, 3) x resident CTAs per SM (default 8, variants 6 and 4), configs 2 and 5
mkdir -p gpurun_out
summ() { python -c "import json,sys;d=json.loads(open(sys.argv[1]).read().strip().splitlines()[-1]);r=d['roofline'];print(sys.argv[2], '%.4g pairs/s  %.3f ms/step  frac %.4f  par %.1e' % (d['value'], d['ms_per_step'], r['frac'], max(d['parity']['u_max_rel'], d['parity']['v_max_rel'])))" "$@"; }
for args in "--config 2 --inv-h 64 --steps 10" "--config 5 --inv-h 128 --path general --steps 5"; do
  for T in 2 3; do
    echo "== $args T=$T"
    timeout 600 python bench.py $args --targets-per-thread $T --no-e2e --no-cpu-baseline > gpurun_out/ft_def.json 2>&1 && summ gpurun_out/ft_def.json "default" || tail -3 gpurun_out/ft_def.json
    for lib in build/variants/*.so; do
      n=$(basename $lib .so)
      STOKES_ER_LIB=$PWD/$lib timeout 600 python bench.py $args --targets-per-thread $T --no-e2e --no-cpu-baseline > gpurun_out/ft_$n.json 2>&1 && summ gpurun_out/ft_$n.json "$n" || tail -3 gpurun_out/ft_$n.json
    done
  done
done
timeout 600 python tools/parity_sweep.py gpurun_out/parity_sweep_t3.json 400 > gpurun_out/parity_sweep_t3.log 2>&1; echo "sweep rc=$?"; tail -2 gpurun_out/parity_sweep_t3.log
