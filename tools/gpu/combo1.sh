# node-path A/B (c-major items vs the s-major build), node-path parity tests, the R20 interpolation study,
# and the treecode MINB=3 variant (config 5 at 1/h = 256)
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_nodes.py -q -x > gpurun_out/pytest_nodes_c1.log 2>&1; echo "nodes tests rc=$?"; tail -2 gpurun_out/pytest_nodes_c1.log
bash tools/gpu/var_nodes.sh
bash tools/gpu/interp_study.sh
summ() { python -c "import json,sys;d=json.loads(open(sys.argv[1]).read().strip().splitlines()[-1]);print(sys.argv[2], '%.4g pairs/s  %.2f ms/step  frac %.4f' % (d['value'], d['ms_per_step'], d['roofline']['frac']), d['config'].get('max_rel_diff_vs_direct'))" "$@"; }
timeout 900 python bench.py --workload tree --config 5 --inv-h 256 --steps 3 --no-cpu-baseline > gpurun_out/tree_def.json 2>&1 && summ gpurun_out/tree_def.json tree_default || tail -3 gpurun_out/tree_def.json
STOKES_ER_LIB=$PWD/build/treevar/libstokes_er_treeminb3.so timeout 900 python bench.py --workload tree --config 5 --inv-h 256 --steps 3 --no-cpu-baseline > gpurun_out/tree_minb3.json 2>&1 && summ gpurun_out/tree_minb3.json tree_minb3 || tail -3 gpurun_out/tree_minb3.json
echo done
