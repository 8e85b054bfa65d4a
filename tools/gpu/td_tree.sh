mkdir -p gpurun_out

timeout 1800 python tools/twodrop_table2.py gpurun_out/twodrop_table2_tree.json 16 32 64 128 256 --tree 2>&1 | grep -v "^ \|^{\|^}\|^\]" | head -20
python -c "
import json;d=json.load(open('gpurun_out/twodrop_table2_tree.json'))
for r in d['rows']: print({k:(round(v,9) if isinstance(v,float) else v) for k,v in r.items() if k in ('inv_h','iterations','solve_ms','max_err','l2_err','order_max','order_l2','max_err_away_0.5','order_away_0.5','tree')})
"
