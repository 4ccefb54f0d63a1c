"""K9 (element matrices) time on c5 vs the threads-per-block knob VB_K9_BLOCK (one fresh process
per setting; the first context of a process pays the module load, so the second is reported)."""
import os, subprocess, sys

code = r'''
import os, sys, time
sys.path.insert(0, os.getcwd())
os.environ["VB_SETUP_TIMES"] = "1"
import torch
import paper_2304_09770_b200 as vb
from synthetic import make_problem
from synthetic.configs import C5_DIMS
prob = make_problem("c5", dims=C5_DIMS[1])
for i in range(2):
    t = time.time(); ctx = vb.context_for(prob); torch.cuda.synchronize(); print("context %.3f" % (time.time() - t), flush=True)
    ctx.close()
'''
for b in sys.argv[1:] or ["128", "64", "32"]:
    env = dict(os.environ, VB_K9_BLOCK=b)
    out = subprocess.run([sys.executable, "-c", code], env=env, capture_output=True, text=True)
    k9 = [l for l in out.stderr.splitlines() + out.stdout.splitlines() if "K9" in l or "context" in l]
    print("VB_K9_BLOCK=%s" % b, *k9, sep="\n  ", flush=True)
