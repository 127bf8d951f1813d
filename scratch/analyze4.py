import sys, numpy as np
sys.path.insert(0,'.')
import oracle as O
g=O.gen('rmat',22,16,1)
p=O.h2_degree_aware(g,1)
key=(p.astype(np.uint64)<<np.uint64(32))|(np.arange(g.n,dtype=np.uint64)+np.uint64(1))
deg=np.diff(g.off)
src=np.repeat(np.arange(g.n),deg)
higher = key[g.nbr] > key[src]
pos_from_end = (g.off[src+1]-1) - np.arange(g.nbr.size)
big=np.int64(1<<40)
first = np.full(g.n, big); np.minimum.at(first, src[higher], pos_from_end[higher])
cand = first==big
exam = np.where(cand, deg, first+1)
nz = deg>0
def cost(steps):
    # steps: list of step sizes, last repeats
    tot_g=0; tot_steps=0
    e=exam[nz]; d=deg[nz]
    covered=np.zeros(e.size,np.int64); nst=np.zeros(e.size,np.int64)
    k=0
    while True:
        st=steps[min(k,len(steps)-1)]
        act = covered < e
        if not act.any(): break
        take = np.minimum(st, d-covered)
        covered = np.where(act, covered+take, covered)
        nst += act
        tot_g += np.where(act, take, 0).sum()
        k+=1
    return tot_g, nst.mean(), np.percentile(nst,99)
for steps in ([4],[2,2,4],[1,3,4],[2,4,8],[1,2,4,8],[8],[1,4,8],[2,6,8]):
    gth, mst, p99 = cost(steps)
    print(steps, 'gathers', gth, 'mean steps', round(mst,2), 'p99 steps', p99)
print('exact examined', exam.sum())
