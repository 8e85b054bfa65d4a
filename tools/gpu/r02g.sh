# final evidence of the re-entry session: r02b.sh (tests, smoke, default/general/two-drop bench lines, launch list,
# sym_kernel capture) + the treecode bench line at 1/h = 256 and a capture of its walk kernel
mkdir -p gpurun_out
TAG=${TAG:-r02g}
TAG=$TAG bash tools/gpu/r02b.sh
timeout 900 python bench.py --workload tree --config 5 --inv-h 256 --steps 3 --no-cpu-baseline > gpurun_out/bench_${TAG}_tree256.json 2> gpurun_out/bench_${TAG}_tree256.err; echo "bench tree rc=$?"
timeout 1200 ncu --section SpeedOfLight --section ComputeWorkloadAnalysis --section WarpStateStats --section Occupancy --section LaunchStats --section InstructionStats \
  --metrics sm__pipe_fp64_cycles_active.avg.pct_of_peak_sustained_active,dram__bytes_read.sum,dram__bytes_write.sum \
  --clock-control none -k regex:"tree_far_kernel" -c 1 -o gpurun_out/tree_$TAG python bench.py --workload tree --config 5 --inv-h 256 --steps 1 --warmup 3 --no-e2e --no-cpu-baseline > gpurun_out/ncu_tree_$TAG.log 2>&1; echo "ncu tree rc=$?"
echo done_g
