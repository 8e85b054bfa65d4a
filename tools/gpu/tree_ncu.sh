mkdir -p gpurun_out
cat > /tmp/tree_one.py <<'PY'
import sys, torch
sys.path.insert(0, '.')
import paper_2507_00156_b200 as ser
from workloads.configs import config5
blk = config5(inv_h=int(sys.argv[1]))
plan = ser.TreePlan(blk.src_xyz, int(sys.argv[2]), int(sys.argv[3]), 0.6)
arrs = ser.to_device(blk)
for _ in range(2):
    ser.evaluate_tree(*arrs, blk.h, blk.rho, plan)
torch.cuda.synchronize()
PY
timeout 300 python /tmp/tree_one.py 128 4000 8 && echo clean-ok
timeout 900 ncu --set full --clock-control none --import-source on -k regex:"tree_far" -c 1 -o gpurun_out/tree_full python /tmp/tree_one.py 128 4000 8 > gpurun_out/tree_ncu.log 2>&1
echo "ncu rc=$?"
