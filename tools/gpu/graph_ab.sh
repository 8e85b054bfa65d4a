# CUDA-graph replay vs eager timing of the bench step (config 1, config 2 at 1/h = 32, config 5 at 1/h = 64 both paths)
mkdir -p gpurun_out
summ() { python -c "import json,sys;d=json.loads(open(sys.argv[1]).read().strip().splitlines()[-1]);r=d['roofline'];p=d['parity'];print(sys.argv[2], '%.4g pairs/s  %.4f ms/step  kernel %.4f ms share %.3f  near %.3f  par %.1e %.1e  launches %s' % (d['value'], d['ms_per_step'], r['kernel_ms'], r['kernel_share'], d.get('near_kernel',{}).get('ms',0), p['u_max_rel'], p['v_max_rel'], d['gpu_launches']))" "$@"; }
timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_gpu_bench.py -q -x > gpurun_out/pytest_graph.log 2>&1; echo "pytest rc=$?"; tail -2 gpurun_out/pytest_graph.log
for args in "--config 1 --inv-h 16 --steps 200" "--config 2 --inv-h 32 --steps 40" "--config 5 --inv-h 64 --steps 20 --path general" "--config 5 --inv-h 64 --steps 20 --path nodes" "--config 2 --inv-h 64 --steps 10 --schedule separate"; do
  for g in off on; do
    timeout 600 python bench.py $args --graph $g --no-e2e --no-cpu-baseline > gpurun_out/g_$g.json 2>&1 && summ gpurun_out/g_$g.json "$args graph=$g" || tail -3 gpurun_out/g_$g.json
  done
done
