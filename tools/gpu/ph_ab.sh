# near-phase cap A/B (SER_MAX_PHASES 64 default vs build/variants): small and mid-size problems
mkdir -p gpurun_out
summ() { python -c "import json,sys;d=json.loads(open(sys.argv[1]).read().strip().splitlines()[-1]);print(sys.argv[2], '%.4g %s  %.4f ms/step' % (d['value'], d['unit'], d['ms_per_step']))" "$@"; }
for args in "--config 1 --inv-h 16 --steps 200" "--config 2 --inv-h 16 --steps 100" "--config 3 --inv-h 16 --steps 100" "--workload twodrop --inv-h 16 --steps 5" "--workload twodrop --inv-h 32 --steps 3" "--config 2 --inv-h 24 --steps 50"; do
  for rep in 1 2; do
  timeout 600 python bench.py $args --no-e2e --no-cpu-baseline > gpurun_out/ph_def.json 2>&1 && summ gpurun_out/ph_def.json "$args default" || tail -3 gpurun_out/ph_def.json
  STOKES_ER_LIB=$PWD/build/variants/libstokes_er_ph128.so timeout 600 python bench.py $args --no-e2e --no-cpu-baseline > gpurun_out/ph_128.json 2>&1 && summ gpurun_out/ph_128.json "$args ph128" || tail -3 gpurun_out/ph_128.json
  done
done
