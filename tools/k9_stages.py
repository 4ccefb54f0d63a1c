"""K9 stage-time experiment (VB_K9_STOP=n ends the element kernel before stage n+1): element
kernel time on c5 for each cut.  Not a benchmark; the results are garbage for n > 0."""
import os
import subprocess
import sys

code = r'''
import os, sys, time
sys.path.insert(0, os.getcwd())
os.environ["VB_SETUP_TIMES"] = "1"
import torch
import paper_2304_09770_b200 as vb
from synthetic import make_problem
from synthetic.configs import C5_DIMS
prob = make_problem(sys.argv[1], dims=C5_DIMS[1] if sys.argv[1] == "c5" else None)
for i in range(2):
    ctx = vb.context_for(prob); ctx.close()
'''
for cfg in sys.argv[1:] or ["c5"]:
    for stop in [1, 2, 3, 5, 6, 8, 0]:   # 8: everything but stage (9)
        env = dict(os.environ, VB_K9_STOP=str(stop), VB_SETUP_TIMES="1", VB_NO_SETUP_OVERLAP="1")
        r = subprocess.run([sys.executable, "-c", code, cfg], env=env, capture_output=True, text=True)
        lines = [l for l in r.stderr.splitlines() if "K9" in l]
        print(cfg, "stop", stop, lines[-1] if lines else r.stderr[-300:], flush=True)
