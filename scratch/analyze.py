import sys, numpy as np, time
sys.path.insert(0,'.')
import oracle as O
t=time.time()
name=sys.argv[1]
if name=='rmat22': g=O.gen('rmat',22,16,1)
elif name=='grid': g=O.gen('grid',4096)
elif name=='rgg': g=O.gen('rgg',24000000,3.0,1)
else: g=O.gen('gnp_avg',100000,16.0,1)
print('gen',time.time()-t)
p=O.h2_degree_aware(g,1)
key=(p.astype(np.uint64)<<np.uint64(32))|(np.arange(g.n,dtype=np.uint64)+np.uint64(1))
deg=np.diff(g.off)
# round 1: all alive. examined-from-end until first higher key
src=np.repeat(np.arange(g.n),deg)
higher = key[g.nbr] > key[src]
# position from end within row
pos_from_end = (g.off[src+1]-1) - np.arange(g.nbr.size)
big=np.int64(1<<40)
first = np.full(g.n, big)
np.minimum.at(first, src[higher], pos_from_end[higher])
cand = first==big
exam = np.where(cand, deg, first+1)
print('n',g.n,'cand',cand.sum(),'isolated',(deg==0).sum())
print('total examined', exam.sum(), 'nnz', g.nbr.size)
for K in (1,2,4,8,16,32):
    dec = exam<=K
    print(f'K={K}: decided in stage A {dec.sum()} ({dec.mean():.3f}); deferred {(~dec).sum()}, deferred examined {(exam[~dec]-K).sum()}, cand deferred {(cand&~dec).sum()}')
for lo,hi in ((5,8),(9,16),(17,32),(33,64),(65,256),(257,1024),(1025,8192),(8193,1<<40)):
    s=(exam>=lo)&(exam<=hi)
    print(f'exam in [{lo},{hi}]: {s.sum()} vertices, entries {exam[s].sum()}, cand {(cand&s).sum()}')
# push-store hotness in round 1
cs = cand[src]
tgt = g.nbr[cs]
print('push stores', tgt.size)
lines = tgt // 128
cnt = np.bincount(lines)
top = np.sort(cnt)[::-1][:10]
print('stores to hottest 128B lines of next[]:', top.tolist())
kl = (tgt // 16)  # key lines (8 B keys, 16 per line)
c2 = np.bincount(g.nbr // 16)
print('gathers (all entries) to hottest key lines:', np.sort(c2)[::-1][:5].tolist())
