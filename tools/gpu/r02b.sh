# round-2 full check: GPU tests, smoke, default bench (node path), general-path and two-drop lines,
# launch list, and a light ncu capture (no SASS-patching sections) of the default bench's dominant kernel
mkdir -p gpurun_out
TAG=${TAG:-r02b}
if [ -z "$SKIP_TESTS" ]; then
timeout 2400 python -m pytest tests -m gpu -q ${PYTEST_ARGS} > gpurun_out/pytest_gpu_$TAG.log 2>&1; echo "pytest rc=$?" >> gpurun_out/pytest_gpu_$TAG.log
tail -4 gpurun_out/pytest_gpu_$TAG.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke_$TAG.log 2>&1; echo "smoke rc=$?" >> gpurun_out/smoke_$TAG.log
tail -5 gpurun_out/smoke_$TAG.log
fi
timeout 900 python bench.py > gpurun_out/bench_$TAG.json 2> gpurun_out/bench_$TAG.err; echo "bench rc=$?"
timeout 900 python bench.py --path general --no-cpu-baseline > gpurun_out/bench_${TAG}_general.json 2> gpurun_out/bench_${TAG}_general.err; echo "bench general rc=$?"
timeout 900 python bench.py --workload twodrop --inv-h 64 --steps 5 > gpurun_out/bench_${TAG}_twodrop64.json 2> gpurun_out/bench_${TAG}_twodrop64.err; echo "bench twodrop rc=$?"
if [ -z "$SKIP_NCU" ]; then
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none -c 60 --csv --log-file gpurun_out/launches_$TAG.csv python bench.py --steps 1 --warmup 3 --no-e2e --no-cpu-baseline > gpurun_out/ncu_launch_$TAG.log 2>&1; echo "ncu launch rc=$?"
timeout 1800 ncu --section SpeedOfLight --section MemoryWorkloadAnalysis --section ComputeWorkloadAnalysis --section WarpStateStats --section Occupancy --section LaunchStats --section SchedulerStats --section InstructionStats \
  --metrics smsp__sass_thread_inst_executed_op_dfma_pred_on.sum,smsp__sass_thread_inst_executed_op_dmul_pred_on.sum,smsp__sass_thread_inst_executed_op_dadd_pred_on.sum,sm__pipe_fp64_cycles_active.avg.pct_of_peak_sustained_active,sm__inst_executed_pipe_fp64.avg.pct_of_peak_sustained_active,dram__bytes_read.sum,dram__bytes_write.sum \
  --clock-control none -k regex:"sym_kernel" -c 1 -o gpurun_out/full_$TAG python bench.py --steps 1 --warmup 3 --no-e2e --no-cpu-baseline > gpurun_out/ncu_full_$TAG.log 2>&1; echo "ncu capture rc=$?"
tail -2 gpurun_out/ncu_full_$TAG.log
fi
echo done
