# config 1 after a prologue change: parity tests of the small path, the bench line, the launch list
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_parity.py -q -x > gpurun_out/pytest_cfg1b.log 2>&1; echo "pytest rc=$?"; tail -2 gpurun_out/pytest_cfg1b.log
timeout 300 python bench.py --config 1 --inv-h 16 --steps 200 --no-e2e --no-cpu-baseline > gpurun_out/c1.json 2>&1
python -c "import json;d=json.loads(open('gpurun_out/c1.json').read().strip().splitlines()[-1]);r=d['roofline'];print('step', d['ms_per_step'], 'kernel', r['kernel_ms'], 'share', r['kernel_share'], 'par', d['parity']['u_max_rel'], d['parity']['v_max_rel'])" || tail -5 gpurun_out/c1.json
ncu --metrics gpu__time_duration.sum --clock-control none -c 40 --csv --log-file gpurun_out/launches_cfg1_cur.csv python bench.py --config 1 --inv-h 16 --steps 5 --warmup 3 --no-e2e --no-cpu-baseline --graph off > gpurun_out/ncu_l.log 2>&1; python tools/launch_summary.py gpurun_out/launches_cfg1_cur.csv
