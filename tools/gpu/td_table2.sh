# PAPER.md Table 2 on one B200 (default geometry, R17): direct to 1/h = 128, treecode to 256
mkdir -p gpurun_out
summ() { python -c "
import json,sys;d=json.load(open(sys.argv[1]));print(d['geometry'])
for r in d['rows']: print({k:(float('%.4g'%v) if isinstance(v,float) else v) for k,v in r.items() if k in ('inv_h','iterations','solve_ms','max_err','l2_err','order_max','order_l2','max_err_away_0.5','order_away_0.5','tree')})
" "$1"; }
timeout 1200 python tools/twodrop_table2.py gpurun_out/twodrop_table2.json 16 32 64 128 > gpurun_out/td2_direct.log 2>&1; echo "direct rc=$?"
summ gpurun_out/twodrop_table2.json
timeout 1800 python tools/twodrop_table2.py gpurun_out/twodrop_table2_tree.json 16 32 64 128 256 --tree > gpurun_out/td2_tree.log 2>&1; echo "tree rc=$?"
summ gpurun_out/twodrop_table2_tree.json
