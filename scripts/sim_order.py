"""Simulate k_classify's best-first dynamics for CTAs formed two ways: Morton (7-bit, point 10) and by the
fiber's box-proxy nearest tile (ties by Morton).  Per CTA: list = union of tiles passing the threshold sphere
bound; order = close-count*256 + passes (current k_cull rule).  Per fiber, walk the list: tile bound with the
live tau (boxes), candidates = centroids passing test1+test2 (3-point score <= tau), evaluated in ascending
3-point score (winner first) with the exact d_ME; count hits (tiles with >= 1 candidate) and full evaluations."""
import sys; import os; _R=os.path.dirname(os.path.dirname(os.path.abspath(__file__))); sys.path.insert(0,os.path.join(_R,'scripts')); sys.path.insert(0,_R)
import tile_eval as t, numpy as np
from synth import atlas_for_config, fibers_for_config
at=atlas_for_config(3); fib_all=fibers_for_config(3); N=len(fib_all)
tb, mem, sph = t.current_plan(at); S=sph.astype(np.float64)
fl=t.canon_flips(at); Cc,_=t.feats(at,fl)
T=len(tb)
blo=np.zeros((T,3,3)); bhi=np.zeros((T,3,3))
for k in range(T):
    m=np.unique(mem[k])
    for qq,pt in enumerate((0,10,20)): blo[k,qq]=Cc[m,pt].min(0); bhi[k,qq]=Cc[m,pt].max(0)
thrT=at.thresh.astype(np.float64)[tb]
C=at.centroids
lo=C.reshape(-1,3).min(0)-at.thresh.max(); hi=C.reshape(-1,3).max(0)+at.thresh.max()
def spread(v):
    v=v&0x3ff; v=(v|(v<<16))&0x030000ff; v=(v|(v<<8))&0x0300f00f; v=(v|(v<<4))&0x030c30c3; v=(v|(v<<2))&0x09249249; return v
q=np.clip(((fib_all[:,10]-lo)*(128/np.maximum(hi-lo,1e-3))).astype(np.int64),0,127)
mkey=spread(q[:,0])|(spread(q[:,1])<<1)|(spread(q[:,2])<<2)
rng=np.random.default_rng(11)
# a random spatial window of fibers: take a contiguous Morton range of 32 CTAs worth, so both compositions see the same fibers
morder=np.argsort(mkey,kind='stable')
while True:
    start=rng.integers(0,N//256-40)*256
    win=morder[start:start+32*256]
    F=fib_all[win].astype(np.float64)
    f0,f10,f20=F[:,0],F[:,10],F[:,20]
    g=F[:256]
    dd=np.sqrt(((g[:,10][:,None]-S[None,:,1,:3])**2).sum(-1)) <= S[None,:,1,3]+thrT[None,:]
    if dd.sum(1).mean() > 5: break
def bd(P,qq):
    d=np.maximum(np.maximum(blo[None,:,qq]-P[:,None],0),P[:,None]-bhi[None,:,qq]); return np.sqrt((d**2).sum(-1))
Db=np.maximum(bd(f10,1), np.minimum(np.maximum(bd(f0,0),bd(f20,2)), np.maximum(bd(f20,0),bd(f0,2))))
near=np.argmin(Db,1)
def passes_thr(idx):
    s=thrT[None,:]+1e-3
    sp=lambda P,qq: np.sqrt(((P[:,None]-S[None,:,qq,:3])**2).sum(-1)) <= S[None,:,qq,3]+s
    g0,g10,g20=f0[idx],f10[idx],f20[idx]
    P=sp(g10,1)&((sp(g0,0)&sp(g20,2))|(sp(g20,0)&sp(g0,2)))
    sc=lambda R: None
    Q=np.sqrt(((g10[:,None]-S[None,:,1,:3])**2).sum(-1))<=S[None,:,1,3]+1e-3
    Q&=((np.sqrt(((g0[:,None]-S[None,:,0,:3])**2).sum(-1))<=S[None,:,0,3]+1e-3)&(np.sqrt(((g20[:,None]-S[None,:,2,:3])**2).sum(-1))<=S[None,:,2,3]+1e-3))|((np.sqrt(((g20[:,None]-S[None,:,0,:3])**2).sum(-1))<=S[None,:,0,3]+1e-3)&(np.sqrt(((g0[:,None]-S[None,:,2,:3])**2).sum(-1))<=S[None,:,2,3]+1e-3))
    return P, P&Q
def simulate(ctas):
    hits=full=0; nf=0; npass=0; nlist=0
    for idx in ctas:
        P,CL=passes_thr(idx)
        listed=np.nonzero(P.any(0))[0]
        nlist+=len(listed)
        pr=CL[:,listed].sum(0)*256+P[:,listed].sum(0)
        order=listed[np.argsort(-pr,kind='stable')]
        for i in idx:
            Fi=F[i]; best=np.inf
            for tt in order:
                tau=min(thrT[tt]**2, best**2)
                s2=(np.sqrt(tau)+1e-3)**2
                # box bound
                def b2(p,qq): d=np.maximum(np.maximum(blo[tt,qq]-p,0),p-bhi[tt,qq]); return (d*d).sum()
                if not (b2(Fi[10],1)<=s2 and ((b2(Fi[0],0)<=s2 and b2(Fi[20],2)<=s2) or (b2(Fi[20],0)<=s2 and b2(Fi[0],2)<=s2))): continue
                npass+=1
                m=np.unique(mem[tt]); Cm=Cc[m]
                m10=((Fi[10]-Cm[:,10])**2).sum(-1)
                rd=np.maximum(m10,np.maximum(((Fi[0]-Cm[:,0])**2).sum(-1),((Fi[20]-Cm[:,20])**2).sum(-1)))
                ri=np.maximum(m10,np.maximum(((Fi[0]-Cm[:,20])**2).sum(-1),((Fi[20]-Cm[:,0])**2).sum(-1)))
                cand=[(rd[k],k,0) for k in range(len(m)) if rd[k]<=tau]+[(ri[k],k,1) for k in range(len(m)) if ri[k]<=tau]
                if not cand: continue
                hits+=1
                cand.sort()
                for sc,k,o in cand:
                    tau=min(thrT[tt]**2, best**2)
                    if sc>tau: continue
                    c=Cm[k] if o==0 else Cm[k][::-1]
                    d2=((Fi-c)**2).sum(-1).max()
                    full+=1
                    if d2<=tau: best=np.sqrt(d2)
            nf+=1
    return hits/nf, full/nf, npass/nf, nlist/len(ctas)
near10=np.argmin(bd(f10,1),1)
o5=np.lexsort((mkey[win], near10))
ctasP=[o5[k*256:(k+1)*256] for k in range(32)]
print("same 8192 fibers, all 32 CTAs of the window")
print("point-10-nearest-tile CTAs: hits/fiber %.3f  full evals/fiber %.3f  box passes/fiber %.2f  listed tiles/CTA %.1f" % simulate(ctasP))
