import sys, warnings, numpy as np
sys.path.insert(0,'.'); sys.path.insert(0,'tests'); warnings.filterwarnings("ignore")
import paper_2204_06204_b200 as B
from oracle import bisimp_oracle as O, approx_inverse_oracle as M
spec=B.problems.l_bracket(48)
for algo in ["mg_pcg","mg_vcycle"]:
    cfg=B.SolverConfig(algorithm=algo,max_iters=40); res=B.run(spec,cfg)
    og=O.build_grid(spec.nx,spec.ny,spec.fixtures,spec.loads); steps=cfg.resolved_inner_steps()
    orc=O.run_loop(og,nx=spec.nx,ny=spec.ny,volume_fraction=spec.volume_fraction,passive_mask=spec.passive_mask(),algorithm=algo,max_iters=40,
        low_level_fn=lambda g,a,u,r: M.low_level(g,a,u,algo,1.0,r,steps))
    c=np.array(res.record.compliance); oc=np.array([r[1] for r in orc["rows"]])
    print(algo, ["%.1e"%x for x in (np.abs(c-oc)/np.maximum(np.abs(oc),1e-300))[:25]])
