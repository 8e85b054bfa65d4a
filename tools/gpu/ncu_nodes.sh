# ncu --set full of the node path's kernels (sym_kernel, nbr_kernel) at 1/h = ${H:-128}, after a clean run
mkdir -p gpurun_out
H=${H:-128}
TAG=${TAG:-nodes_h$H}
timeout 600 python bench.py --inv-h $H --steps 3 --no-e2e --no-cpu-baseline > gpurun_out/pre_$TAG.json 2>&1 || { echo "pre-run failed"; tail -20 gpurun_out/pre_$TAG.json; exit 1; }
timeout ${NCU_TIMEOUT:-1500} ncu --set full --clock-control none --import-source on -k regex:"${KREGEX:-sym_kernel|nbr_kernel}" -c ${NCU_COUNT:-2} -o gpurun_out/full_$TAG python bench.py --inv-h $H --steps 1 --warmup 3 --no-e2e --no-cpu-baseline > gpurun_out/ncu_full_$TAG.log 2>&1
echo "ncu rc=$?"
tail -3 gpurun_out/ncu_full_$TAG.log
