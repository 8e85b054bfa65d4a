# one ncu --set full capture of the pair kernel (after a clean run)
mkdir -p gpurun_out
TAG=${TAG:-cur}
timeout 300 python bench.py --steps 3 --no-e2e --no-cpu-baseline $BENCH_ARGS > gpurun_out/pre_$TAG.json 2>&1 || exit 1
timeout 900 ncu --set full --clock-control none --import-source on -k regex:"${KREGEX:-pair_kernel|fused_kernel|far_kernel|near_kernel}" -c ${NCU_COUNT:-1} -o gpurun_out/full_$TAG python bench.py --steps 1 --warmup 3 --no-e2e --no-cpu-baseline $BENCH_ARGS > gpurun_out/ncu_full_$TAG.log 2>&1
echo "ncu rc=$?"
