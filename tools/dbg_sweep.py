import sys; sys.path.insert(0,'.')
import numpy as np, torch, hmg_inputs as hi, oracle
from paper_1605_00492_b200 import Hierarchy
for (ref,nz) in [(2,64),(4,64),(2,16),(2,32),(2,40),(3,128)]:
    cfg=hi.Config('d',ref,ref,nz,0.01,1e-4); lam,b=hi.make_inputs(cfg)
    g=Hierarchy(ref,ref,nz,0.01,1e-4,lam); o=oracle.Hierarchy(ref,ref,nz,0.01,1e-4,lam)
    u0=hi.uniform_vector(b.shape,3)
    for ns,zero in ((1,True),(1,False)):
        u=g.to_device(ref,u0); g.line_smooth(ref,g.to_device(ref,b),u,ns,0.8,zero)
        got=g.to_host(ref,u); refv=o.sweep(ref,b,None if zero else u0,ns,0.8)
        bad=np.argwhere(got!=refv)
        cols=np.unique(bad[:,1]); ks=np.unique(bad[:,0])
        print(ref,nz,ns,zero,'nbad',len(bad),'cols',cols[:10],len(cols),'ks',ks[:5],ks[-3:] if len(ks) else None)
