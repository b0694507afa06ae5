import sys, time; import os; sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import paper_1603_08081_b200 as fb
from paper_1603_08081_b200.configs import CONFIGS, approx_of, spatial_of, image_of
from oracle.pyoracle import Oracle
O=Oracle()
print('fma peak', fb.probe_fma_peak())
for name in ['c1','c3','c2']:
    c=CONFIGS[name]; img=image_of(c); s=spatial_of(c); a=approx_of(c)
    for v in ['fused','naive']:
        t=time.time(); g=fb.bilateral_fast(img,s,a,variant=v,check_epsilon=c.check_epsilon); dt=time.time()-t
        rows=(0, min(64,c.height))
        ref,rc,_=O.bilateral_fast(img,s.profile,s.radius,s.w0,a.d,a.omega,a.max_pointwise_error,c.check_epsilon,rows[0],rows[1],8)
        print(name, v, 'maxabs', np.abs(g[rows[0]:rows[1]]-ref).max(), 'time', dt, flush=True)
