# quadratic-Newton rsqrt in the symmetric kernel: seed accuracy probe, node-path parity with the variant, A/B at 1/h = 256
mkdir -p gpurun_out
./tools/probes/rsqrt_seed_probe > gpurun_out/rsqrt_seed_probe.txt 2>&1; cat gpurun_out/rsqrt_seed_probe.txt
STOKES_ER_LIB=$PWD/build/variants/libstokes_er_rsq2.so timeout 600 python -m pytest tests/test_gpu_nodes.py -q -x > gpurun_out/rsq2_nodes_tests.log 2>&1; tail -3 gpurun_out/rsq2_nodes_tests.log
summ() { python -c "import json,sys;d=json.loads(open(sys.argv[1]).read().strip().splitlines()[-1]);r=d['roofline'];p=d['parity'];print(sys.argv[2], '%.4g pairs/s  %.2f ms/step  frac %.4f  u %.2e v %.2e' % (d['value'], d['ms_per_step'], r['frac'], p['u_max_rel'], p['v_max_rel']))" "$@"; }
for rep in 1 2; do
  timeout 300 python bench.py --steps 3 --no-e2e --no-cpu-baseline > gpurun_out/rq_def.json 2>&1 && summ gpurun_out/rq_def.json default
  STOKES_ER_LIB=$PWD/build/variants/libstokes_er_rsq2.so timeout 300 python bench.py --steps 3 --no-e2e --no-cpu-baseline > gpurun_out/rq_rsq2.json 2>&1 && summ gpurun_out/rq_rsq2.json rsq2
done 2>&1 | tee gpurun_out/rsq2_ab.log
