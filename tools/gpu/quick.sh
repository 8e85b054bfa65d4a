# quick GPU iteration: gpu tests + bench (both schedules), no profiler
mkdir -p gpurun_out
timeout 900 python -m pytest tests -m gpu -x -q > gpurun_out/pytest_gpu.log 2>&1; echo "pytest rc=$?" >> gpurun_out/pytest_gpu.log
tail -3 gpurun_out/pytest_gpu.log
for sch in fused separate; do
  timeout 600 python bench.py --schedule $sch --no-e2e --no-cpu-baseline > gpurun_out/bench_$sch.json 2> gpurun_out/bench_$sch.err
  echo "$sch rc=$?"; python -c "import json;d=json.load(open('gpurun_out/bench_$sch.json'));print(d['value'],d['ms_per_step'],d['roofline']['kernel_ms'],d['roofline']['frac'])"
done
