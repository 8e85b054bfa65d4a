# config 1 (small problem) A/B: default library vs build/variants/*.so, and near-phase overrides
mkdir -p gpurun_out
summ() { python -c "import json,sys;d=json.loads(open(sys.argv[1]).read().strip().splitlines()[-1]);r=d['roofline'];p=d['parity'];print(sys.argv[2], '%.4g pairs/s  %.4f ms/step  kernel %.4f ms share %.3f  par %.1e %.1e' % (d['value'], d['ms_per_step'], r['kernel_ms'], r['kernel_share'], p['u_max_rel'], p['v_max_rel']))" "$@"; }
timeout 900 python -m pytest tests/test_gpu_parity.py -q -x -k "config1 or small_sort or ragged or empty or degenerate" > gpurun_out/pytest_cfg1.log 2>&1; echo "pytest rc=$?"; tail -2 gpurun_out/pytest_cfg1.log
for ph in 0 16 32 64 128 256; do
  timeout 300 python bench.py --config 1 --inv-h 16 --steps 200 --near-phases $ph --no-e2e --no-cpu-baseline > gpurun_out/c1_def.json 2>&1 && summ gpurun_out/c1_def.json "default ph=$ph" || tail -3 gpurun_out/c1_def.json
  for lib in build/variants/*.so; do
    n=$(basename $lib .so)
    STOKES_ER_LIB=$PWD/$lib timeout 300 python bench.py --config 1 --inv-h 16 --steps 200 --near-phases $ph --no-e2e --no-cpu-baseline > gpurun_out/c1_$n.json 2>&1 && summ gpurun_out/c1_$n.json "$n ph=$ph" || tail -3 gpurun_out/c1_$n.json
  done
done
