# sym_kernel study: per-SM active-cycle balance (1/h = 128, 256) and one --set full capture with source (1/h = 64)
mkdir -p gpurun_out
for H in 128 256; do
  timeout 900 ncu --metrics sm__cycles_active.avg,sm__cycles_active.max,sm__cycles_active.min,gpu__time_duration.sum,sm__pipe_fp64_cycles_active.avg.pct_of_peak_sustained_active,sm__pipe_fp64_cycles_active.max.pct_of_peak_sustained_active --clock-control none -k regex:sym_kernel -c 1 --csv python bench.py --inv-h $H --path nodes --steps 1 --warmup 3 --no-e2e --no-cpu-baseline > gpurun_out/sym_balance_h$H.csv 2> gpurun_out/sym_balance_h$H.err
  echo "balance h$H rc=$?"; grep -v "^==" gpurun_out/sym_balance_h$H.csv | tail -8
done
timeout 900 ncu --set full --clock-control none --import-source on -k regex:sym_kernel -c 1 -o gpurun_out/sym_src_h64 python bench.py --inv-h 64 --path nodes --steps 1 --warmup 3 --no-e2e --no-cpu-baseline > gpurun_out/sym_src_h64.log 2>&1
echo "full rc=$?"; tail -2 gpurun_out/sym_src_h64.log
