mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_treecode.py -x -q 2>&1 | tail -1
timeout 600 python tools/tree_scaling.py gpurun_out/ts_default.json 128 256 2>&1 | python -c "
import sys
for l in sys.stdin:
    if l.startswith('{'):
        d=eval(l); print('default', d['inv_h'], d['N0'], d['p'], round(d['direct_ms'],1), round(d['tree_ms'],1), round(d['speedup'],2))"
for lib in build/variants/*.so; do
  n=$(basename $lib .so)
  STOKES_ER_LIB=$PWD/$lib timeout 600 python tools/tree_scaling.py gpurun_out/ts_$n.json 128 256 2>&1 | python -c "
import sys
for l in sys.stdin:
    if l.startswith('{'):
        d=eval(l); print('$n', d['inv_h'], d['N0'], d['p'], round(d['direct_ms'],1), round(d['tree_ms'],1), round(d['speedup'],2))"
done
