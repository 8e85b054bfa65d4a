# treecode: fused near units (default) vs split (SER_TREE_FUSED_NEAR=0: no spills in the walk) at config 5,
# then a light ncu capture of the walk kernel at 1/h = 256 for the library given by TREE_LIB (default: in-tree)
mkdir -p gpurun_out
summ() { python -c "import json,sys;d=json.loads(open(sys.argv[1]).read().strip().splitlines()[-1]);print(sys.argv[2], '%.4g pairs/s  %.2f ms/step  frac %.4f diff %s' % (d['value'], d['ms_per_step'], d['roofline']['frac'], d['config'].get('max_rel_diff_vs_direct')))" "$@"; }
for H in 128 256; do
  for rep in 1 2; do
  timeout 900 python bench.py --workload tree --config 5 --inv-h $H --steps 3 --no-cpu-baseline > gpurun_out/tree_def_h$H.json 2>&1 && summ gpurun_out/tree_def_h$H.json "fused h$H" || tail -3 gpurun_out/tree_def_h$H.json
  STOKES_ER_LIB=$PWD/build/treevar/libstokes_er_tsplit.so timeout 900 python bench.py --workload tree --config 5 --inv-h $H --steps 3 --no-cpu-baseline > gpurun_out/tree_split_h$H.json 2>&1 && summ gpurun_out/tree_split_h$H.json "split h$H" || tail -3 gpurun_out/tree_split_h$H.json
  done
done
LIBENV=""
if [ -n "$TREE_LIB" ]; then LIBENV="STOKES_ER_LIB=$PWD/$TREE_LIB"; fi
env $LIBENV timeout 1500 ncu --section SpeedOfLight --section ComputeWorkloadAnalysis --section WarpStateStats --section Occupancy --section LaunchStats --section MemoryWorkloadAnalysis \
  --metrics sm__pipe_fp64_cycles_active.avg.pct_of_peak_sustained_active,dram__bytes_read.sum,dram__bytes_write.sum \
  --clock-control none -k regex:"tree_far_kernel|near_kernel" -c 2 -o gpurun_out/full_tree_h256 python bench.py --workload tree --config 5 --inv-h 256 --steps 1 --warmup 1 --no-cpu-baseline > gpurun_out/ncu_tree_h256.log 2>&1; echo "ncu rc=$?"
echo done
