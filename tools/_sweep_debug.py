import numpy as np, sys, os
sys.path.insert(0,'/root/repo'); sys.path.insert(0,'/root/repo/tests')
from helpers import gpu_scores, oracle_scores, scheme_of
from paper_2205_07610_b200 import _native as N
ctx=N.Context(0)
rng=np.random.default_rng(5)
sch=scheme_of((2,-1,2,1),'affine')
for L in list(range(1,40))+[50,64,65,100,150]:
    q=[rng.integers(0,4,L).astype(np.uint8) for _ in range(2)]
    s=[rng.integers(0,4,min(L,64)).astype(np.uint8) for _ in range(2)]
    pairs=[(0,0),(1,1)]
    got=gpu_scores(ctx,q,s,pairs,sch,'local','f16x2'); want=oracle_scores(q,s,pairs,sch,'local')
    ok=all((got[k]==want[k]).all() for k in range(3))
    if not ok: print(L, "got",[ (int(got[0][i]),int(got[1][i]),int(got[2][i])) for i in range(2)],"want",[(int(want[0][i]),int(want[1][i]),int(want[2][i])) for i in range(2)])
print("done")
