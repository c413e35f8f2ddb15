"""Seed quality offline (cfg 3, 4,000 sampled fibers, final keys from the oracle cache): how often the
best-first winner of the nearest tile(s) under several nearness criteria is the fiber's final best."""
import sys
import os; sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import importlib.util
spec = importlib.util.spec_from_file_location("te", os.path.join(os.path.dirname(os.path.abspath(__file__)), 'tile_eval.py')); te = importlib.util.module_from_spec(spec); spec.loader.exec_module(te)
from synth import atlas_for_config, fibers_for_config, sample_indices
EPS=1e-3
at = atlas_for_config(3)
fl = te.canon_flips(at); Cc, F = te.feats(at, fl)
tb, mem, sph = te.current_plan(at); S=sph.astype(np.float64); T=len(tb)
thr=at.thresh.astype(np.float64); R=S[:,:,3]+thr[tb][:,None]+EPS
z=np.load(os.path.join(os.path.dirname(os.path.dirname(os.path.abspath(__file__))), 'cache', 'oracle', 'cfg3_exact.npz')); dist=z['dist'].astype(np.float64); lab=z['label']
idx=sample_indices(4145000, 4000, seed=9)
fib=fibers_for_config(3)[idx].astype(np.float64)
dfin=np.where(lab[idx]>=0, dist[idx], np.inf)
C=Cc  # canonical centroids (orientation canonical)
def dme2(f, m):  # f [21,3], m centroid ids -> min over orientation of max sq dist
    a=((f[None]-C[m])**2).sum(-1).max(-1); b=((f[None,::-1]-C[m])**2).sum(-1).max(-1); return np.minimum(a,b)
res={k:[] for k in ('nearest','near2','near3','d10','lb','ub','mid')}
for i in range(len(fib)):
    f=fib[i]; p0,p10,p20=f[0],f[10],f[20]
    d10=((p10-S[:,1,:3])**2).sum(-1); d00=((p0-S[:,0,:3])**2).sum(-1); d2020=((p20-S[:,2,:3])**2).sum(-1)
    d020=((p0-S[:,2,:3])**2).sum(-1); d200=((p20-S[:,0,:3])**2).sum(-1)
    r0,r10,r20=R[:,0]**2,R[:,1]**2,R[:,2]**2
    pas=(d10<=r10)&(((d00<=r0)&(d2020<=r20))|((d020<=r20)&(d200<=r0)))
    dc=np.maximum(d10,np.minimum(np.maximum(d00,d2020),np.maximum(d020,d200)))
    dc=np.where(pas,dc,np.inf)
    order=np.argsort(dc)
    def seed_of(tiles):
        best=np.inf
        for t in tiles:
            if not np.isfinite(dc[t]): continue
            m=mem[t]; thr2=thr[tb[t]]**2
            # 3-point score
            def sc3(fa):
                return np.maximum.reduce([((fa[0]-C[m,0])**2).sum(-1),((fa[10]-C[m,10])**2).sum(-1),((fa[20]-C[m,20])**2).sum(-1)])
            s=np.minimum(np.where(sc3(f)<=thr2,sc3(f),np.inf),np.where(sc3(f[::-1])<=thr2,sc3(f[::-1]),np.inf))
            k=np.argmin(s)
            if not np.isfinite(s[k]): continue
            d=dme2(f,np.array([m[k]]))[0]
            if d<=thr2: best=min(best,d)
        return best
    res['nearest'].append(seed_of(order[:1]))
    res['near2'].append(seed_of(order[:2]))
    res['near3'].append(seed_of(order[:3]))
    o10=np.argsort(np.where(pas,d10,np.inf)); res['d10'].append(seed_of(o10[:1]))
    sq=lambda x: np.sqrt(x)
    rr0,rr10,rr20=S[:,0,3],S[:,1,3],S[:,2,3]
    lb=np.maximum(sq(d10)-rr10, np.minimum(np.maximum(sq(d00)-rr0, sq(d2020)-rr20), np.maximum(sq(d020)-rr20, sq(d200)-rr0)))
    ub=np.maximum(sq(d10)+rr10, np.minimum(np.maximum(sq(d00)+rr0, sq(d2020)+rr20), np.maximum(sq(d020)+rr20, sq(d200)+rr0)))
    mid=np.maximum(sq(d10)+0.5*rr10, np.minimum(np.maximum(sq(d00)+0.5*rr0, sq(d2020)+0.5*rr20), np.maximum(sq(d020)+0.5*rr20, sq(d200)+0.5*rr0)))
    res['lb'].append(seed_of(np.argsort(np.where(pas,lb,np.inf))[:1]))
    res['ub'].append(seed_of(np.argsort(np.where(pas,ub,np.inf))[:1]))
    res['mid'].append(seed_of(np.argsort(np.where(pas,mid,np.inf))[:1]))
fin2=dfin**2
for k,v in res.items():
    if not v: continue
    v=np.array(v); lab_ok=np.isfinite(fin2)
    exact=np.isclose(v,fin2,rtol=1e-6)&lab_ok
    print(f"{k:8s} seeded {np.isfinite(v).mean():.3f}  seed==final {exact.sum()/lab_ok.sum():.3f}  mean ratio(seed/final, both finite) {np.nanmean(np.where(np.isfinite(v)&lab_ok, v/np.where(fin2>0,fin2,1), np.nan)):.3f}")
