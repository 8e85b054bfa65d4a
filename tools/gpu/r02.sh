# round-2 check on the B200: GPU tests, smoke, default bench (config 5, 1/h = 256), launch list and
# one ncu --set full capture of the dominant kernel for the SAME bench configuration
mkdir -p gpurun_out
TAG=${TAG:-r02}
if [ -z "$SKIP_TESTS" ]; then
timeout 1500 python -m pytest tests -m gpu -x -q ${PYTEST_ARGS} > gpurun_out/pytest_gpu_$TAG.log 2>&1; echo "pytest rc=$?" >> gpurun_out/pytest_gpu_$TAG.log
tail -3 gpurun_out/pytest_gpu_$TAG.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke_$TAG.log 2>&1; echo "smoke rc=$?" >> gpurun_out/smoke_$TAG.log
cat gpurun_out/smoke_$TAG.log
fi
timeout 900 python bench.py $BENCH_ARGS > gpurun_out/bench_$TAG.json 2> gpurun_out/bench_$TAG.err; echo "bench rc=$?"
cat gpurun_out/bench_$TAG.json | head -c 600; echo
if [ -z "$SKIP_NCU" ]; then
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none -c 60 --csv --log-file gpurun_out/launches_$TAG.csv python bench.py --steps 1 --warmup 3 --no-e2e --no-cpu-baseline $BENCH_ARGS > gpurun_out/ncu_launch_$TAG.log 2>&1; echo "ncu launch rc=$?"
timeout 1200 ncu --set full --clock-control none --import-source on -k regex:"${KREGEX:-fused_kernel|far_kernel|sym_|near_kernel}" -c 1 -o gpurun_out/full_$TAG python bench.py --steps 1 --warmup 3 --no-e2e --no-cpu-baseline $BENCH_ARGS > gpurun_out/ncu_full_$TAG.log 2>&1; echo "ncu full rc=$?"
fi
echo done
