mkdir -p gpurun_out
for H in 128 256; do
  timeout 900 python bench.py --workload onsurface --inv-h $H --steps 3 > gpurun_out/bench_onsurface_h$H.json 2> gpurun_out/bench_onsurface_h$H.err; echo "onsurface h$H rc=$?"
  python -c "import json,sys;d=json.loads(open(sys.argv[1]).read().strip().splitlines()[-1]);print(sys.argv[1], '%.4g pairs/s %.2f ms frac %.3f path %s diff %s' % (d['value'], d['ms_per_step'], d['roofline']['frac'], d['config']['path'], d['config'].get('max_rel_diff_vs_oracle_sample')))" gpurun_out/bench_onsurface_h$H.json
done
timeout 1200 python tools/twodrop_table2.py gpurun_out/twodrop_table2_r02.json 16 32 64 128 > gpurun_out/td_table2_r02.log 2>&1; echo "table2 rc=$?"
timeout 900 python -m pytest tests/test_gpu_bench.py -q > gpurun_out/pytest_bench_c5.log 2>&1; echo "bench tests rc=$?"; tail -2 gpurun_out/pytest_bench_c5.log
