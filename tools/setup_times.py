import os, sys, time
sys.path.insert(0, os.getcwd())
os.environ["VB_SETUP_TIMES"] = "1"
import torch
import paper_2304_09770_b200 as vb
from synthetic import make_problem
from synthetic.configs import C5_DIMS
t = time.time(); prob = make_problem("c5", dims=C5_DIMS[1]); print("make_problem %.3f" % (time.time() - t), flush=True)
for i in range(2):
    t = time.time(); ctx = vb.context_for(prob); torch.cuda.synchronize(); print("context %.3f" % (time.time() - t), flush=True)
    ctx.close()
