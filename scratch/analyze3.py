import sys, numpy as np
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
big=np.int64(1<<40)
while alive.any():
    rnd+=1
    kcur=np.where(alive,key,np.uint64(0))
    higher = (kcur[g.nbr] > kcur[src]) & alive[src]
    first=np.full(g.n,big); np.minimum.at(first, src[higher], pos_from_end[higher])
    cand = alive & (first==big)
    nonc = alive & ~cand
    hit = cand[g.nbr] & nonc[src]
    f2=np.full(g.n,big); np.minimum.at(f2, src[hit], pos_from_end[hit])
    removed = nonc & (f2<big)
    surv = nonc & ~removed
    pull_exam = np.where(removed, f2+1, 0) + np.where(surv, deg, 0)
    push = deg[cand].sum()
    print(f'round {rnd}: alive {alive.sum()} cand {cand.sum()} removed {removed.sum()} surv {surv.sum()} | push stores {push} | pull examined {pull_exam.sum()} (removed part {np.where(removed,f2+1,0).sum()}, survivors {deg[surv].sum()}) max pull row {pull_exam.max()}')
    alive = surv
