"""CPU model (diagnostics): per-brick iteration counts of Jacobi-PCG against additive coarse
corrections on 8^3 (AG) aggregates — exact coarse solve (add2) and k damped-Jacobi coarse sweeps
(j1..j4) — on the level-0 bricks of an N^3 two-level phantom hierarchy, float64, stop ||r|| <= 1e-6
||b||, with the error against the tol-1e-10 oracle.  The basis of the brick engine's coarse
correction (csrc/rwb_resident4.cu).   Usage: python tools/brick_cc_model.py [N] [AG] [S1|S2] [bricks]
"""
import sys, itertools; sys.path.insert(0,'/root/repo')
import numpy as np
from oracle import rw as orw, lod
from paper_2509_26213_b200 import synthetic
N=int(sys.argv[1]) if len(sys.argv)>1 else 128
AG=int(sys.argv[2]) if len(sys.argv)>2 else 8
which=sys.argv[3] if len(sys.argv)>3 else "S1"
shape=(N,)*3; B=32
vol=synthetic.phantom(shape); seeds=synthetic.seeds(shape,which)
P=orw.RWParams(tol=1e-10)
vols=lod.lod_chain(vol,(B,)*3,2); s1=orw.project_seeds(seeds)
top=orw.solve_level(vols[1],s1,vols[1].shape,None,orw.RWParams(tol=1e-8))
bound=orw.upsample_linear(top.prob,shape)
bid,nb=orw.brick_ids(shape,(B,)*3)
S=orw.assemble(vol,seeds,bid,nb,bound,P)
x_ref,_,_=orw.pcg(S,bound,orw.RWParams(tol=1e-10))
def sl3(a,k): 
    o=[slice(None)]*3; o[k]=a; return tuple(o)
res=[]
rng=np.random.default_rng(1)
ids=list(range(nb)); rng.shuffle(ids)
for b in ids[:int(sys.argv[4]) if len(sys.argv)>4 else 16]:
    bz,by,bx=np.unravel_index(b,(N//B,)*3)
    sl=(slice(bz*B,bz*B+B),slice(by*B,by*B+B),slice(bx*B,bx*B+B))
    unk=S.unknown[sl]; d=np.where(unk,S.diag[sl],1.0); s=np.where(unk,1/np.sqrt(d),0)
    W=[]
    for k in range(3):
        w=S.coupled[k][sl].copy(); last=[slice(None)]*3; last[k]=slice(B-1,B); w[tuple(last)]=0
        a=sl3(slice(0,-1),k); bb=sl3(slice(1,None),k)
        ws=np.zeros_like(w); ws[a]=w[a]*s[a]*s[bb]; W.append(ws)
    def A(x):
        y=x*unk
        for k in range(3):
            a=sl3(slice(0,-1),k); bb=sl3(slice(1,None),k)
            y[a]-=W[k][a]*x[bb]; y[bb]-=W[k][a]*x[a]
        return y
    x0=np.where(unk,bound[sl],0)/np.where(unk,s,1)*unk
    rhs=S.rhs[sl]*s
    # aggregates AGxAGxAG
    na=B//AG
    agg=lambda v: v.reshape(na,AG,na,AG,na,AG).sum((1,3,5))
    Pm=lambda xc: xc.repeat(AG,0).repeat(AG,1).repeat(AG,2)*unk
    # coarse operator A_c = P^T A P
    nc=na**3; Ac=np.zeros((nc,nc))
    for j in range(nc):
        e=np.zeros(nc); e[j]=1; Ac[:,j]=agg(A(Pm(e.reshape(na,na,na)))).ravel()
    live=np.diag(Ac)>0
    Ac[~live,:]=0; Ac[:,~live]=0; Ac[~live,~live]=1
    Aci=np.linalg.inv(Ac)
    dci=1/np.diag(Ac)
    def coarse(r): return Pm((Aci@agg(r).ravel()).reshape(na,na,na))
    def coarse_j(r,k,om=0.8):
        g=agg(r).ravel(); c=om*dci*g
        for _ in range(k-1): c=c+om*dci*(g-Ac@c)
        return Pm(c.reshape(na,na,na))
    precs={"jacobi":lambda r:r,"add2":lambda r:r+coarse(r),"j1":lambda r:r+coarse_j(r,1),"j2":lambda r:r+coarse_j(r,2),"j3":lambda r:r+coarse_j(r,3),"j4":lambda r:r+coarse_j(r,4)}
    out=[b]
    bb2=(rhs**2).sum()
    for nm,pr in precs.items():
        y=x0.copy(); r=rhs-A(y); z=pr(r); p=z.copy(); rz=(r*z).sum(); it=0
        while (r*r).sum()>1e-12*bb2 and it<5000:
            q=A(p); al=rz/(p*q).sum(); y+=al*p; r-=al*q; z=pr(r); rzn=(r*z).sum(); p=z+rzn/rz*p; rz=rzn; it+=1
        err=np.abs(np.where(unk,y*s,0)-np.where(unk,x_ref[sl],0)).max()
        out+= [nm,it,f"{err:.1e}"]
    print(*out,flush=True)
