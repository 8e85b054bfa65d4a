# A/B of the default library against build/variants/*.so on the node path (config 5), 1/h = 128 twice, 256 once
mkdir -p gpurun_out
summ() { python -c "import json,sys;d=json.loads(open(sys.argv[1]).read().strip().splitlines()[-1]);r=d['roofline'];print(sys.argv[2], '%.4g pairs/s  %.3f ms/step  frac %.4f  kernel %.2f ms  nbr %.2f ms  par %.1e' % (d['value'], d['ms_per_step'], r['frac'], r['kernel_ms'], d.get('near_kernel',{}).get('ms',0), max(d['parity']['u_max_rel'], d['parity']['v_max_rel'])))" "$@"; }
run() {
  args="$1"
  echo "== $args"
  timeout 600 python bench.py $args --no-e2e --no-cpu-baseline > gpurun_out/vn_def.json 2>&1 && summ gpurun_out/vn_def.json "default" || tail -3 gpurun_out/vn_def.json
  for lib in build/variants/*.so; do
    n=$(basename $lib .so)
    STOKES_ER_LIB=$PWD/$lib timeout 600 python bench.py $args --no-e2e --no-cpu-baseline > gpurun_out/vn_$n.json 2>&1 && summ gpurun_out/vn_$n.json "$n" || tail -3 gpurun_out/vn_$n.json
  done
}
run "--inv-h 128 --path nodes --steps 10"
run "--inv-h 128 --path nodes --steps 10"
[ -z "$SKIP256" ] && run "--inv-h 256 --steps 2"
