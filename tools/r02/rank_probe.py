import sys; sys.path[:0]=['.','oracle']
import numpy as np, paper_2001_04321_b200 as P, pyoracle as O
gen=np.random.default_rng(1)
for shape,r in (([40,30,20],100),([60,50,40],128),([30,20,10,8],80)):
    t=gen.random(shape); m=[gen.random((d,r)) for d in shape]
    prov=P.GpuDenseProvider(t)
    try:
        errs=[float(np.linalg.norm(prov.mttkrp(m,k)-O.mttkrp(t,m,k))/np.linalg.norm(O.mttkrp(t,m,k))) for k in range(len(shape))]
        print(shape,r,"mttkrp rel err",errs, [prov.mttkrp_plan(r,k)[:30] for k in range(len(shape))])
    except Exception as e:
        print(shape,r,"ERR",type(e).__name__,str(e)[:200])
    prov.close()
