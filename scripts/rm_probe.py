import sys, numpy as np
sys.path.insert(0, '/root/repo')
sys.path.insert(0, '/root/repo/tests')
import paper_2007_12623_b200 as ss
from conftest import load_golden
g = load_golden("tex_d16")
p = g["params"]
rd, rv = ss.refine_disparities(g["clean_disp"], g["clean_valid"], g["left"], g["right"], p)
print("mismatch", int((rd.view(np.uint32) != g["refine_disp"].view(np.uint32)).sum()), int((rv != g["refine_valid"]).sum()))
