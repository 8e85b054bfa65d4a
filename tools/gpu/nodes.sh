# node-target path: its GPU tests first, then bench lines, then the whole GPU suite
mkdir -p gpurun_out
TAG=${TAG:-nodes}
timeout 900 python -m pytest tests/test_gpu_nodes.py -x -q > gpurun_out/pytest_nodes_$TAG.log 2>&1; echo "pytest nodes rc=$?" >> gpurun_out/pytest_nodes_$TAG.log
tail -3 gpurun_out/pytest_nodes_$TAG.log
for H in 64 128 256; do
  timeout 600 python bench.py --inv-h $H --no-cpu-baseline > gpurun_out/bench_${TAG}_h$H.json 2> gpurun_out/bench_${TAG}_h$H.err; echo "bench h$H rc=$?"
done
if [ -z "$SKIP_SUITE" ]; then
timeout 1800 python -m pytest tests -m gpu -q > gpurun_out/pytest_gpu_$TAG.log 2>&1; echo "pytest rc=$?" >> gpurun_out/pytest_gpu_$TAG.log
tail -5 gpurun_out/pytest_gpu_$TAG.log
fi
echo done
