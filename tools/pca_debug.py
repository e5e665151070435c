import sys; sys.path.insert(0,'.')
import numpy as np, torch
import paper_2505_15511_b200 as nb
from oracle import Oracle
o=Oracle("port"); ctx=nb.Context(0)
for (n,d,b) in [(3000,24,8),(700,33,3),(2000,200,5)]:
    x=o.gaussian_mixture(n,d,b,10.0,23)
    e=nb.pca_init(x,9,ctx=ctx); f=nb.pca_init(x,9,ctx=ctx,fast=True); f2=nb.pca_init(x,9,ctx=ctx,fast=True)
    print(n,d,b,"fast-fast",float(abs(f-f2).max()),"fast-exact",float(abs(f-e).max()),
          "corr", np.corrcoef(e[:,0],f[:,0])[0,1], np.corrcoef(e[:,1],f[:,1])[0,1], np.corrcoef(e[:,0],f[:,1])[0,1])
    print(" e", e[:3].tolist()); print(" f", f[:3].tolist())
    xt=torch.tensor(x,dtype=torch.float64,device='cuda'); xc=xt-xt.mean(0); C=(xc.T@xc/n)
    ev=torch.linalg.eigvalsh(C).flip(0)[:4]; print(" eig", ev.tolist())
