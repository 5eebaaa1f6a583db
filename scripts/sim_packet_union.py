"""Packet-union simulation (design aid, CPU; not product or test code): for 10^6
uniform 3D points in Morton order, the mean number of points within the packet's query
box dilated by the largest exact 10-th-NN distance among its queries — for packets of
32 consecutive positions and for tree-aligned packets (maximal canonical subtrees of at
most 32 points).  Printed numbers are quoted in DESIGN.md §12.0."""
import numpy as np, sys
sys.path.insert(0,'/root/repo')
import zdgen
from scipy.spatial import cKDTree
n=1_000_000
pts=zdgen.uniform(n,3,seed=3).astype(np.int64)
def spread(v):
    k=np.zeros_like(v,dtype=np.uint64)
    for b in range(21):
        k |= ((v>>b)&1).astype(np.uint64) << np.uint64(3*b)
    return k
key=(spread(pts[:,0])<<np.uint64(2))|(spread(pts[:,1])<<np.uint64(1))|spread(pts[:,2])
o=np.lexsort((np.arange(n),key)); P=pts[o].astype(np.float64); K=key[o]
T=cKDTree(P)
d,_=T.query(P,k=11); rk=d[:,10]
# tree-aligned packets: maximal canonical subtrees with <= 32 points
packets=[]; stack=[(0,n)]
Kl=[int(x) for x in K]
while stack:
    lo,hi=stack.pop()
    if hi-lo<=32 or Kl[lo]==Kl[hi-1]:
        packets.append((lo,hi)); continue
    b=(Kl[lo]^Kl[hi-1]).bit_length()-1
    # split point: first index with bit b set
    import bisect
    pref=(Kl[lo]>>(b+1))<<(b+1); mid=bisect.bisect_left(Kl,pref|(1<<b),lo,hi)
    stack.append((lo,mid)); stack.append((mid,hi))
sizes=np.array([h-l for l,h in packets])
print("tree packets",len(packets),"mean size",sizes.mean(),"lane util",sizes.mean()/32)
rng=np.random.default_rng(0)
def union(lo,hi):
    Q=P[lo:hi]; lo3=Q.min(0); hi3=Q.max(0); b=rk[lo:hi].max()
    cand=T.query_ball_point((lo3+hi3)/2, np.sqrt((((hi3-lo3)/2)**2).sum())+b)
    C=P[cand]; g=np.maximum(np.maximum(lo3-C,C-hi3),0); return ((np.sqrt((g**2).sum(1)))<=b).sum()
sel=rng.choice(len(packets),3000,replace=False)
U=[union(*packets[i]) for i in sel]; S=[sizes[i] for i in sel]
print("tree-aligned: mean union",np.mean(U),"per query",np.sum(U)/np.sum(S), "per lane-slot(32)", np.mean(U))
sel2=rng.choice(n//32,3000,replace=False)
U2=[union(i*32,i*32+32) for i in sel2]
print("consecutive-32: mean union",np.mean(U2),"per query",np.mean(U2)/32)
