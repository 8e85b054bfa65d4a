mkdir -p gpurun_out
for v in def tr2; do
  if [ $v = tr2 ]; then export STOKES_ER_LIB=$PWD/build/variants/libstokes_er_tr2.so; fi
  timeout 900 ncu --section SpeedOfLight --section WarpStateStats --section SchedulerStats --section InstructionStats --section SourceCounters --import-source on \
    --metrics sm__pipe_fp64_cycles_active.avg.pct_of_peak_sustained_active,smsp__sass_thread_inst_executed_op_dfma_pred_on.sum,smsp__sass_thread_inst_executed_op_dmul_pred_on.sum,smsp__sass_thread_inst_executed_op_dadd_pred_on.sum \
    --clock-control none -k regex:"sym_kernel" -c 1 -o gpurun_out/sym_$v python bench.py --inv-h 64 --path nodes --steps 1 --warmup 1 --no-e2e --no-cpu-baseline > gpurun_out/ncu_sym_$v.log 2>&1; echo "$v rc=$?"
done
