import sys, torch
sys.path.insert(0, '.')
import paper_2507_00156_b200 as ser
from workloads.twodrop import twodrop
s = ser.twodrop_solver(twodrop(64))
s.solve(); torch.cuda.synchronize()
PY=1
