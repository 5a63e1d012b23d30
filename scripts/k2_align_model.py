"""Offline model for profiles/r2_k2_align_ab.txt: distinct 128-byte lines per
K2 quad gather instruction (8u x 4v warps, c4 geometry, cell reuse) for the
lock-step and the plane-aligned lane schedules.  Usage: python k2_align_model.py
[view angle in rad]."""
import numpy as np, sys
rng=np.random.default_rng(0)
N=512; sp=0.5; org=-(N-1)/2*sp  # centered voxel centres
nu,nv,du,dv=1248,960,0.64,0.64
SID,SDD=750.,1200.
step=0.25
nxp=nyp=N+4
def rays(theta, iu, iv):
    S=np.array([SID*np.cos(theta),SID*np.sin(theta),0.])
    er=S/SID; et=np.array([-np.sin(theta),np.cos(theta),0.]); ez=np.array([0,0,1.])
    D=S[None]-SDD*er[None]+((iu-(nu-1)/2)*du)[:,None]*et[None]+((iv-(nv-1)/2)*dv)[:,None]*ez[None]
    d=D-S; d/=np.linalg.norm(d,axis=1,keepdims=True)
    return S,d
def clip(S,d):
    lo=org-0.5*sp; hi=org+(N-0.5)*sp
    with np.errstate(divide='ignore',invalid='ignore'):
        ta=(lo-S[None])/d; tb=(hi-S[None])/d
    t0=np.nanmax(np.minimum(ta,tb),axis=1); t1=np.nanmin(np.maximum(ta,tb),axis=1)
    return t0,t1
def warp_cost(theta, u0, v0, align):
    iu=u0+np.tile(np.arange(8),4); iv=v0+np.repeat(np.arange(4),8)
    S,d=rays(theta,iu.astype(float),iv.astype(float))
    t0,t1=clip(S,d); hit=t1>t0
    if not hit.any(): return 0,0,0
    n=np.where(hit,np.ceil((t1-t0)/step),0).astype(int)
    dt=np.where(hit,(t1-t0)/np.maximum(n,1),0)
    xdom=abs(d[0,0])>abs(d[0,1])
    p0=(S[None]+(t0+0.5*dt)[:,None]*d-org)/sp+2
    dd=dt[:,None]*d/sp
    dom=0 if xdom else 1
    if align:
        # lanes start so their first samples sit on a common dominant plane
        pd=p0[:,dom]; ddd=dd[:,dom]
        ref=np.where(hit, pd, np.nan)
        # plane reached first along direction of travel
        sgn=np.sign(np.nanmean(ddd[hit]))
        start_plane=np.nanmin(ref*sgn)*sgn
        s=np.where(hit,np.round((pd-start_plane)/ddd),0).astype(int)
        s=np.maximum(s,0)
    else:
        s=np.zeros(32,int)
    iters=int((s+n).max())
    lines=0; samples=int(n.sum()); loads=0
    prev=np.full(32,-1)
    for i in range(iters):
        k=i-s; act=hit&(k>=0)&(k<n)
        if not act.any(): continue
        p=p0+k[:,None]*dd
        c=np.floor(p).astype(np.int64)
        if xdom: off=c[:,2]*nxp*nyp+c[:,0]*nyp+c[:,1]
        else: off=c[:,2]*nxp*nyp+c[:,1]*nxp+c[:,0]
        ld=act&(off!=prev)
        prev=np.where(act,off,prev)
        if ld.any():
            lines+=len(np.unique((off[ld]*16)//128)); loads+=ld.sum()
    return lines,samples,loads,iters
theta=float(sys.argv[1]) if len(sys.argv)>1 else 0.5
tot={False:[0,0,0,0],True:[0,0,0,0]}
for w in range(300):
    u0=8*rng.integers(0,nu//8); v0=4*rng.integers(0,nv//4)
    for al in (False,True):
        r=warp_cost(theta,u0,v0,al)
        if r[0]==0: continue
        for j in range(4): tot[al][j]+=r[j]
for al in (False,True):
    L,Sm,ld,it=tot[al]
    print('align' if al else 'plain', 'lines/sample %.3f'%(L/Sm), 'loads/sample %.3f'%(ld/Sm), 'lines/load-instr-lane %.3f'%(L/ld*32/4), 'iters/sample*32 %.3f'%(it*32/Sm))
