import sys; sys.path.insert(0,'.')
import numpy as np
import paper_2505_15511_b200 as nb
from oracle import Oracle
o=Oracle("port"); ctx=nb.Context(0)
x=o.gaussian_mixture(700,33,3,10.0,23)
print("exact", file=sys.stderr); e=nb.pca_init(x,9,ctx=ctx)
print("fast", file=sys.stderr); f=nb.pca_init(x,9,ctx=ctx,fast=True)
X=x.astype(np.float64); Xc=X-X.mean(0); w,V=np.linalg.eigh(Xc.T@Xc/700); print("numpy top eig", w[::-1][:3], "v0", V[:2,-1], V[:2,-2], file=sys.stderr)
