mkdir -p gpurun_out
timeout 1800 python -m pytest tests/test_gpu_parity.py tests/test_gpu_nodes.py tests/test_gpu_bench.py -q -x > gpurun_out/pytest_c4.log 2>&1; echo "pytest rc=$?"; tail -3 gpurun_out/pytest_c4.log
timeout 600 python bench.py --config 1 --steps 40 > gpurun_out/bench_c4_cfg1.json 2> gpurun_out/bench_c4_cfg1.err; echo "bench rc=$?"
python -c "import json,sys;d=json.loads(open(sys.argv[1]).read().strip().splitlines()[-1]);r=d['roofline'];print(sys.argv[1], '%.4g pairs/s %.3f ms frac %.3f share %.3f launches %s clocks %s par %s' % (d['value'], d['ms_per_step'], r['frac'], r['kernel_share'], d['gpu_launches'], d['clocks']['samples'], d['parity']['u_max_rel']))" gpurun_out/bench_c4_cfg1.json
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none -c 40 --csv --log-file gpurun_out/launches_cfg1_c4.csv python bench.py --config 1 --steps 2 --warmup 3 --no-e2e --no-cpu-baseline > /dev/null 2>&1; echo "ncu rc=$?"
echo done
