# node tests + AoS/SoA A/B on the node path + small-config bench lines (config 1, config 2 at 1/h = 32)
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_nodes.py -q -x > gpurun_out/pytest_nodes_c2.log 2>&1; echo "nodes tests rc=$?"; tail -2 gpurun_out/pytest_nodes_c2.log
bash tools/gpu/var_nodes.sh
for a in "--config 1" "--config 2 --inv-h 32"; do
  n=$(echo $a | tr -d ' -')
  timeout 600 python bench.py $a --steps 40 > gpurun_out/bench_c2_$n.json 2> gpurun_out/bench_c2_$n.err; echo "bench $a rc=$?"
  python -c "import json,sys;d=json.loads(open(sys.argv[1]).read().strip().splitlines()[-1]);r=d['roofline'];print(sys.argv[1], '%.4g pairs/s %.3f ms frac %.3f share %.3f T %s items %s clocks %s par %s' % (d['value'], d['ms_per_step'], r['frac'], r['kernel_share'], d['config']['targets_per_thread'], d['config']['work_items'], d['clocks']['samples'], d['parity']['u_max_rel']))" gpurun_out/bench_c2_$n.json
done
echo done
