import sys; sys.path.insert(0, ".")
import numpy as np, torch, synth, sys
sys.path.insert(0,'.')
from oracle import discretize as D, mlgmres, fwi
from paper_1703_09268_b200 import api
from tests.helpers import to_dev, to_host, rel
for make in [synth.tiny2d, synth.tiny3d, synth.cfg1]:
    p=make(); w=2*np.pi*p.freqs[0]; pml=D.default_pml(p.m)
    op=api.helm_setup(api.Grid.of(p),p.m,w,api.Pml(pml.R,pml.power,pml.v_ref),api.C128,max_rhs=2)
    hier=mlgmres.Hierarchy(p,w,pml)
    b=synth.random_complex((2,p.n_ext),1)
    z=torch.zeros(2,p.n_ext,dtype=torch.complex128,device='cuda')
    api.helm_vcycle(op,to_dev(b),z)
    zg=to_host(z)
    ref=[mlgmres.vcycle(hier,0,b[r]) for r in range(2)]
    print(p.name,[rel(zg[r],ref[r]) for r in range(2)])
    # residual-only check: one smoother
    for l in range(len(hier.shapes)):
        pass
