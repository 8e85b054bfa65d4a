mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_treecode.py -x -q 2>&1 | tail -2
timeout 1500 python tools/tree_scaling.py gpurun_out/tree_scaling.json ${LEVELS:-128 256} 2>&1 | tail -14 | cut -c1-330
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/tree_launches.csv python tools/tree_scaling.py /dev/null 128 > /dev/null 2>&1
python tools/launch_summary.py gpurun_out/tree_launches.csv > gpurun_out/tree_launches.txt; head -12 gpurun_out/tree_launches.txt
