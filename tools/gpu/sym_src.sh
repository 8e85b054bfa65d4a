# one --set full capture with source of sym_kernel at 1/h = 64 (node path)
mkdir -p gpurun_out
timeout 900 ncu --set full --clock-control none --import-source on -k regex:sym_kernel -c 1 -o gpurun_out/sym_src_${TAG:-t3}_h64 python bench.py --inv-h 64 --path nodes --steps 1 --warmup 3 --no-e2e --no-cpu-baseline > gpurun_out/sym_src_${TAG:-t3}_h64.log 2>&1
echo "full rc=$?"
