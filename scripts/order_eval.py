import sys; import os; _R=os.path.dirname(os.path.dirname(os.path.abspath(__file__))); sys.path.insert(0,os.path.join(_R,'scripts')); sys.path.insert(0,_R)
import tile_eval as t, numpy as np
import oracle
from synth import atlas_for_config, fibers_for_config
at=atlas_for_config(3)
fib_all=fibers_for_config(3)
N=len(fib_all)
# Morton 7-bit key of point 10 over the atlas box grown by max thr (as seg_create)
C=at.centroids
lo=C.reshape(-1,3).min(0)-at.thresh.max(); hi=C.reshape(-1,3).max(0)+at.thresh.max()
q=np.clip(((fib_all[:,10]-lo)*(128/np.maximum(hi-lo,1e-3))).astype(np.int64),0,127)
def spread(v):
    v=v&0x3ff; v=(v|(v<<16))&0x030000ff; v=(v|(v<<8))&0x0300f00f; v=(v|(v<<4))&0x030c30c3; v=(v|(v<<2))&0x09249249; return v
key=spread(q[:,0])|(spread(q[:,1])<<1)|(spread(q[:,2])<<2)
order=np.argsort(key,kind='stable')
tb, mem, sph = t.current_plan(at); S=sph.astype(np.float64)
fl=t.canon_flips(at); Cc,_=t.feats(at,fl)
T=len(tb)
blo=np.zeros((T,3,3)); bhi=np.zeros((T,3,3))
for k in range(T):
    m=np.unique(mem[k])
    for qq,pt in enumerate((0,10,20)): blo[k,qq]=Cc[m,pt].min(0); bhi[k,qq]=Cc[m,pt].max(0)
# member -> tile
tile_of=np.zeros(at.M,int)
for k in range(T):
    for m in np.unique(mem[k]): tile_of[m]=k
thr=at.thresh.astype(np.float64)[tb]
rng=np.random.default_rng(3)
ctas=rng.choice(N//256, 12, replace=False)
res={'sphere':[], 'vote-centre':[], 'vote-box':[], 'soft-box':[]}
for cta in ctas:
    idx=order[cta*256:(cta+1)*256]; F=fib_all[idx].astype(np.float64)
    r=oracle.classify(F.astype(np.float32), at.centroids, at.bundle_id, at.thresh, want_d2b=False)
    # best centroid: brute force d_ME for labelled fibers only
    lab=r['label']; ok=lab>=0
    f0,f10,f20=F[:,0],F[:,10],F[:,20]
    s=thr[None,:]+1e-3
    sp=lambda P,qq,R: np.sqrt(((P[:,None]-S[None,:,qq,:3])**2).sum(-1)) <= S[None,:,qq,3]+R
    tb3s=lambda R: sp(f10,1,R)&((sp(f0,0,R)&sp(f20,2,R))|(sp(f20,0,R)&sp(f0,2,R)))
    PASS=tb3s(s)
    CLOSE_S=tb3s(np.full_like(s,1e-3))
    def ib(P,qq): return np.all((P[:,None]>=blo[None,:,qq]-1e-3)&(P[:,None]<=bhi[None,:,qq]+1e-3),-1)
    CLOSE_B=PASS&ib(f10,1)&((ib(f0,0)&ib(f20,2))|(ib(f20,0)&ib(f0,2)))
    listed=np.nonzero(PASS.any(0))[0]
    npass=PASS[:,listed].sum(0)
    # proxies of each fiber's distance to each listed tile
    def bd(P,qq):
        d=np.maximum(np.maximum(blo[None,listed,qq]-P[:,None],0),P[:,None]-bhi[None,listed,qq]); return np.sqrt((d**2).sum(-1))
    def cd(P,qq): return np.sqrt(((P[:,None]-S[None,listed,qq,:3])**2).sum(-1))
    Db=np.maximum(bd(f10,1), np.minimum(np.maximum(bd(f0,0),bd(f20,2)), np.maximum(bd(f20,0),bd(f0,2))))
    Dc=np.maximum(cd(f10,1), np.minimum(np.maximum(cd(f0,0),cd(f20,2)), np.maximum(cd(f20,0),cd(f0,2))))
    Db=np.where(PASS[:,listed], Db, np.inf); Dc=np.where(PASS[:,listed], Dc, np.inf)
    valid=np.isfinite(Db).any(1)
    if len(listed)==0 or not valid.any(): continue
    vb=np.bincount(np.argmin(Db[valid],1), minlength=len(listed)); vc=np.bincount(np.argmin(Dc[valid],1), minlength=len(listed))
    soft=(1.0/(1.0+np.where(np.isfinite(Db),Db,1e9))).sum(0)
    pr={'sphere':CLOSE_S[:,listed].sum(0)*256+npass,
        'vote-centre':vc*65536+CLOSE_S[:,listed].sum(0)*256+npass,
        'vote-box':vb*65536+CLOSE_S[:,listed].sum(0)*256+npass,
        'soft-box':soft}
    # each labelled fiber's best tile: brute force over centroids of its label's bundle
    best_tile=-np.ones(256,int)
    for i in np.nonzero(ok)[0]:
        ms=np.nonzero(at.bundle_id==lab[i])[0]
        Cm=at.centroids[ms].astype(np.float64)
        d=np.minimum(np.sqrt(((F[i]-Cm)**2).sum(-1)).max(1), np.sqrt(((F[i]-Cm[:,::-1])**2).sum(-1)).max(1))
        best_tile[i]=tile_of[ms[np.argmin(d)]]
    for k,v in pr.items():
        ordl=listed[np.argsort(-v,kind='stable')]
        pos={tt:j for j,tt in enumerate(ordl)}
        res[k]+= [pos.get(bt,-1) for bt in best_tile[ok]]
for k,v in res.items():
    v=np.array(v); v=v[v>=0]
    print(f"{k:11s}: best tile's position in the CTA order: mean {v.mean():.2f} median {np.median(v):.0f} first {np.mean(v==0):.3f} top3 {np.mean(v<3):.3f}")
