# final round-2 validation: r02b.sh (tests, smoke, bench lines, launch list, light sym capture) + a full
# capture of the separate-schedule near kernel (config 2, 1/h = 64) for the per-near-pair FP64 counts
mkdir -p gpurun_out
TAG=${TAG:-r02d} bash tools/gpu/r02b.sh
TAG=${TAG:-r02d}
timeout 600 python bench.py --config 2 --inv-h 64 --schedule separate --steps 3 --no-e2e --no-cpu-baseline > gpurun_out/pre_near_$TAG.json 2>&1
timeout 900 ncu --set full --clock-control none --import-source on -k regex:"near_kernel|far_kernel" -c 2 -o gpurun_out/full_near_$TAG python bench.py --config 2 --inv-h 64 --schedule separate --steps 1 --warmup 3 --no-e2e --no-cpu-baseline > gpurun_out/ncu_near_$TAG.log 2>&1; echo "ncu near rc=$?"
echo done2
