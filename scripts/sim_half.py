"""Offline: dense steps per fiber with 32-centroid tiles vs 16-centroid half tiles processed two fibers per
step (max of the two halves' passing fibers per warp), on Morton windows at the final cutoff (cfg 3)."""
import sys
import os; sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import importlib.util
spec = importlib.util.spec_from_file_location("te", os.path.join(os.path.dirname(os.path.abspath(__file__)), 'tile_eval.py')); te = importlib.util.module_from_spec(spec); spec.loader.exec_module(te)
from synth import atlas_for_config, fibers_for_config
EPS=1e-3
at = atlas_for_config(3)
fl = te.canon_flips(at); Cc, F = te.feats(at, fl)
tb, mem, sph = te.current_plan(at)
T=len(tb)
def halves(m):
    m=np.unique(m)
    if len(m)<=16: return [m, m[:0]]
    ext=F[m].max(0)-F[m].min(0); d=int(np.argmax(ext))
    o=np.argsort(F[m,d],kind='stable'); return [m[o[:16]], m[o[16:]]]
def box(ms):
    if len(ms)==0: return np.full((3,3),np.inf), np.full((3,3),-np.inf)
    return np.stack([Cc[ms,p].min(0) for p in (0,10,20)]), np.stack([Cc[ms,p].max(0) for p in (0,10,20)])
full_lo=np.zeros((T,3,3)); full_hi=np.zeros((T,3,3)); h_lo=np.zeros((2,T,3,3)); h_hi=np.zeros((2,T,3,3))
for t in range(T):
    full_lo[t],full_hi[t]=box(np.unique(mem[t]))
    for k,h in enumerate(halves(mem[t])): h_lo[k,t],h_hi[k,t]=box(h)
thr2=(at.thresh.astype(np.float64)**2)[tb]
z=np.load(os.path.join(os.path.dirname(os.path.dirname(os.path.abspath(__file__))), 'cache', 'oracle', 'cfg3_exact.npz')); dist=z['dist'].astype(np.float64); lab=z['label']
dfin=np.where(lab>=0,dist,np.inf)
Fb=fibers_for_config(3)
P0,P10,P20=Fb[:,0].astype(np.float64),Fb[:,10].astype(np.float64),Fb[:,20].astype(np.float64)
del Fb
C10=at.centroids[:,10].astype(np.float64); lo,hi=C10.min(0),C10.max(0)
q=np.clip((P10-lo)/(hi-lo)*127,0,127).astype(np.int64)
def spread3(v):
    v=v.astype(np.uint64); out=np.zeros_like(v)
    for b in range(10): out|=((v>>np.uint64(b))&np.uint64(1))<<np.uint64(3*b)
    return out
key=spread3(q[:,0])|(spread3(q[:,1])<<np.uint64(1))|(spread3(q[:,2])<<np.uint64(2))
order=np.argsort(key,kind='stable')
rng=np.random.default_rng(3); wins=rng.choice(len(order)//256,300,replace=False)
def bp(P,L,H,q):
    d=np.maximum(np.maximum(L[None,:,q]-P[:,None],P[:,None]-H[None,:,q]),0); return (d**2).sum(-1)
now=new=unionh=0
for w in wins:
    idx=order[w*256:(w+1)*256]
    tau=np.minimum(thr2[None],dfin[idx,None]**2); s2=(np.sqrt(tau)+EPS)**2
    def test(L,H):
        return (bp(P10[idx],L,H,1)<=s2)&(((bp(P0[idx],L,H,0)<=s2)&(bp(P20[idx],L,H,2)<=s2))|((bp(P20[idx],L,H,0)<=s2)&(bp(P0[idx],L,H,2)<=s2)))
    pf=test(full_lo,full_hi); pa=test(h_lo[0],h_hi[0]); pb=test(h_lo[1],h_hi[1])
    for wp in range(8):
        sel=np.arange(wp,256,8)
        now+=pf[sel].sum(); new+=np.maximum(pa[sel].sum(0),pb[sel].sum(0)).sum(); unionh+=(pa[sel]|pb[sel]).sum()
print("steps now (full box)",now/len(wins)/256,"per fiber; half-pairs max",new/len(wins)/256,"; union of halves",unionh/len(wins)/256, "ratio", new/now)
