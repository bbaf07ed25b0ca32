"""Ad-hoc GPU debugging helper: sweep small cases against the oracle."""
import sys, os
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np, torch
import inputs, oracle
from paper_1608_04431_b200 import fa

def run(seed, H, W, tile, pnd, pnf):
    d = inputs.random_dirs(seed, H, W, p_nodata=pnd, p_noflow=pnf)
    exp = oracle.accumulate(d)
    try:
        with fa.Context(0, tile=tile) as ctx:
            got = ctx.accumulate(dirs=torch.from_numpy(d).cuda(), atype="u64").cpu().numpy()
        bad = np.flatnonzero((got != exp).ravel())
        return f"mismatch {bad.size}" if bad.size else "ok"
    except fa.FaError as e:
        return str(e)

for case in [(2,300,1,(7,1),0.1,0.0),(2,300,1,(0,0),0.1,0.0),(2,300,1,(64,1),0.1,0.0),(2,14,1,(7,1),0.1,0.0),
             (2,300,1,(7,1),0.0,0.0),(3,300,2,(7,2),0.1,0.0),(2,1,300,(1,7),0.1,0.0),(5,64,64,(0,0),0.0,0.0),(5,70,70,(0,0),0.0,0.0)]:
    print(case, run(*case))
