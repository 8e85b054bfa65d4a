# two-drop solve at 1/h = 64 (self blocks: sym_kernel<2> through the node path) vs symmetric-kernel warp counts
mkdir -p gpurun_out
summ() { python -c "import json,sys;d=json.loads(open(sys.argv[1]).read().strip().splitlines()[-1]);print(sys.argv[2], '%.4g %s  %.2f ms/solve' % (d['value'], d['unit'], d['ms_per_step']))" "$@"; }
for rep in 1 2; do
timeout 900 python bench.py --workload twodrop --inv-h 64 --steps 3 --no-e2e --no-cpu-baseline > gpurun_out/tdw_def.json 2>&1 && summ gpurun_out/tdw_def.json default || tail -3 gpurun_out/tdw_def.json
for lib in build/variants/*.so; do n=$(basename $lib .so)
STOKES_ER_LIB=$PWD/$lib timeout 900 python bench.py --workload twodrop --inv-h 64 --steps 3 --no-e2e --no-cpu-baseline > gpurun_out/tdw_$n.json 2>&1 && summ gpurun_out/tdw_$n.json $n || tail -3 gpurun_out/tdw_$n.json
done; done
ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv --log-file gpurun_out/td64_launch.csv python bench.py --workload twodrop --inv-h 64 --steps 1 --warmup 1 --no-e2e --no-cpu-baseline > /dev/null 2>&1
STOKES_ER_LIB=$PWD/build/variants/libstokes_er_w16.so ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv --log-file gpurun_out/td64_launch_w16.csv python bench.py --workload twodrop --inv-h 64 --steps 1 --warmup 1 --no-e2e --no-cpu-baseline > /dev/null 2>&1
python tools/launch_summary.py gpurun_out/td64_launch.csv | head -12; python tools/launch_summary.py gpurun_out/td64_launch_w16.csv | head -12
