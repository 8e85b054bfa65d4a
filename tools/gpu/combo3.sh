# GPU suite + smoke after the small-problem prologue; config 1 line; fused treecode capture at config 5 1/h=256
mkdir -p gpurun_out
timeout 2400 python -m pytest tests -m gpu -q > gpurun_out/pytest_gpu_c3.log 2>&1; echo "pytest rc=$?" >> gpurun_out/pytest_gpu_c3.log; tail -4 gpurun_out/pytest_gpu_c3.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke_c3.log 2>&1; echo "smoke rc=$?"; tail -4 gpurun_out/smoke_c3.log
for a in "--config 1" "--config 2 --inv-h 32"; do
  n=$(echo $a | tr -d ' -')
  timeout 600 python bench.py $a --steps 40 > gpurun_out/bench_c3_$n.json 2> gpurun_out/bench_c3_$n.err; echo "bench $a rc=$?"
  python -c "import json,sys;d=json.loads(open(sys.argv[1]).read().strip().splitlines()[-1]);r=d['roofline'];print(sys.argv[1], '%.4g pairs/s %.3f ms frac %.3f share %.3f launches %s clocks %s par %s' % (d['value'], d['ms_per_step'], r['frac'], r['kernel_share'], d['gpu_launches'], d['clocks']['samples'], d['parity']['u_max_rel']))" gpurun_out/bench_c3_$n.json
done
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none -c 40 --csv --log-file gpurun_out/launches_cfg1.csv python bench.py --config 1 --steps 2 --warmup 3 --no-e2e --no-cpu-baseline > /dev/null 2>&1; echo "ncu cfg1 launches rc=$?"
timeout 1500 ncu --section SpeedOfLight --section ComputeWorkloadAnalysis --section WarpStateStats --section Occupancy --section LaunchStats --section MemoryWorkloadAnalysis \
  --metrics sm__pipe_fp64_cycles_active.avg.pct_of_peak_sustained_active,dram__bytes_read.sum,dram__bytes_write.sum \
  --clock-control none -k regex:"tree_far_kernel" -c 1 -o gpurun_out/full_tree_fused_h256 python bench.py --workload tree --config 5 --inv-h 256 --steps 1 --warmup 1 --no-cpu-baseline > gpurun_out/ncu_tree_fused_h256.log 2>&1; echo "ncu tree rc=$?"
echo done
