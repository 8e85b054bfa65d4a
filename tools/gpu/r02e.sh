# round-2 re-entry check: GPU tests, smoke, the driver's default bench command
mkdir -p gpurun_out
timeout 1200 python -m pytest tests -m gpu -x -q > gpurun_out/pytest_gpu_e.log 2>&1; echo "pytest rc=$?" >> gpurun_out/pytest_gpu_e.log
tail -3 gpurun_out/pytest_gpu_e.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke_e.log 2>&1; echo "smoke rc=$?"; tail -5 gpurun_out/smoke_e.log
timeout 900 python bench.py > gpurun_out/bench_default_e.json 2> gpurun_out/bench_default_e.err; echo "bench rc=$?"
tail -c 3000 gpurun_out/bench_default_e.json
