import sys, numpy as np, time
sys.path.insert(0,'.')
import oracle as O
name=sys.argv[1]
if name=='rmat22': g=O.gen('rmat',22,16,1)
elif name=='grid': g=O.gen('grid',4096)
elif name=='rgg': g=O.gen('rgg',24000000,3.0,1)
else: g=O.gen('gnp_avg',100000,16.0,1)
p=O.h2_degree_aware(g,1)
key=(p.astype(np.uint64)<<np.uint64(32))|(np.arange(g.n,dtype=np.uint64)+np.uint64(1))
deg=np.diff(g.off)
src=np.repeat(np.arange(g.n),deg)
pos_from_end = (g.off[src+1]-1) - np.arange(g.nbr.size)
alive=np.ones(g.n,bool)
rnd=0
while alive.any():
    rnd+=1
    kcur=np.where(alive,key,np.uint64(0))
    higher = (kcur[g.nbr] > kcur[src]) & alive[src]
    big=np.int64(1<<40)
    first=np.full(g.n,big); np.minimum.at(first, src[higher], pos_from_end[higher])
    cand = alive & (first==big)
    exam = np.where(cand, deg, first+1); exam[~alive]=0
    A=alive
    print(f'round {rnd}: alive {A.sum()} cand {cand.sum()} examined {exam.sum()} nnz(A) {deg[A].sum()} max_exam {exam.max()} nnz(C) {deg[cand].sum()} max deg cand {deg[cand].max() if cand.any() else 0}')
    for lo,hi in ((33,256),(257,4096),(4097,1<<40)):
        s=(exam>=lo)&(exam<=hi)
        print(f'   exam in [{lo},{hi}]: {s.sum()} vertices, entries {exam[s].sum()}, cand {(cand&s).sum()}')
    # update
    X=np.zeros(g.n,bool); X[g.nbr[cand[src]]]=True
    alive = alive & ~cand & ~X
