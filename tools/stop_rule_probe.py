"""CPU probe (diagnostics): is a whole-level miss of the 1e-4 bar the solver's or the stop rule's?

Rebuilds case N of tools/random_parity.py (same generator), assembles the Jacobi-scaled system
the device solves, and runs Jacobi-PCG and the masked-aggregation V-cycle PCG of rwb_mgcg.cu in
numpy, in float64 and float32, with the device's stop rule ||r|| <= 1e-7 ||S b||, against the
tol-1e-10 oracle.  Case 2 ((175, 100), one level): every variant stops with the same 3.4e-3 error
(an unseeded pocket whose value the residual cannot see), i.e. the miss is the stop rule's.
Usage: python tools/stop_rule_probe.py [case] [strength threshold]
"""
import sys, itertools; sys.path.insert(0,'/root/repo')
import numpy as np
from oracle import rw as orw
from paper_2509_26213_b200 import synthetic
rng = np.random.default_rng(7)
target=int(sys.argv[1]) if len(sys.argv)>1 else 2
TH=float(sys.argv[2]) if len(sys.argv)>2 else 0.01
for case in range(target+1):
    if case % 3 == 2:
        shape = tuple(int(rng.integers(70, 200)) for _ in range(2)); brick = (64, 64)
    else:
        shape = tuple(int(rng.integers(33, 100)) for _ in range(3)); brick = (32, 32, 32)
    levels = int(rng.integers(1, 3))
    vol = synthetic.phantom(shape) + 0.05 * rng.standard_normal(shape).astype(np.float32)
    vol = np.clip(vol, 0, 1).astype(np.float32)
    seeds = synthetic.seeds(shape, "S1" if case % 2 else "S2")
print(case, shape, levels)
P=orw.RWParams(tol=1e-10)
ref=orw.solve_level(vol,seeds,shape,None,P).prob
v3=vol.reshape((1,)*(3-vol.ndim)+vol.shape); s3=seeds.reshape(v3.shape); shape3=v3.shape
bid,nb=orw.brick_ids(shape3,shape3)
S=orw.assemble(v3,s3,bid,nb,None,P)
unk=S.unknown
s=np.where(unk,1/np.sqrt(S.diag),0.0)
W=[np.zeros(shape3) for _ in range(3)]
for k in range(3):
    a=orw._sl(3,k,slice(0,-1)); b=orw._sl(3,k,slice(1,None))
    W[k][a]=S.coupled[k][a]*s[a]*s[b]
def Aop(W,dg,x):
    y=dg*x
    for k in range(3):
        a=orw._sl(3,k,slice(0,-1)); b=orw._sl(3,k,slice(1,None))
        y[a]-=W[k][a]*x[b]; y[b]-=W[k][a]*x[a]
    return y
def faces(W):
    f=np.zeros(W[0].shape)
    for k in range(3):
        a=orw._sl(3,k,slice(0,-1)); b=orw._sl(3,k,slice(1,None))
        f[a]+=W[k][a]; f[b]+=W[k][a]
    return f
dg0=unk.astype(float); leak0=np.where(unk,1.0-faces(W),0.0)
def strong_mask(W,dg):
    sh=dg.shape; m=np.zeros(sh,bool)
    Z,Y,X=[(n+1)//2 for n in sh]
    for A in itertools.product(range(Z),range(Y),range(X)):
        cells=[(2*A[0]+a,2*A[1]+b,2*A[2]+c) for a in (0,1) for b in (0,1) for c in (0,1)]
        cells=[c for c in cells if all(c[k]<sh[k] for k in range(3)) and dg[c]>0]
        if not cells: continue
        par={c:c for c in cells}
        def f(c):
            while par[c]!=c: c=par[c]
            return c
        for c in cells:
            for k in range(3):
                d=list(c); d[k]+=1; d=tuple(d)
                if d in par and W[k][c]>=TH*min(dg[c],dg[d]): par[f(c)]=f(d)
        comps={}
        for c in cells: comps.setdefault(f(c),[]).append(c)
        best=max(comps.values(),key=len)
        for c in best: m[c]=True
    return m
def agg(v,sh):
    pad=[(0,2*c-n) for c,n in zip(sh,v.shape)]
    v=np.pad(v,pad); return v.reshape(sh[0],2,sh[1],2,sh[2],2).sum((1,3,5))
def coarsen(W,leak,dg):
    m=strong_mask(W,dg); sh=tuple((n+1)//2 for n in leak.shape)
    lk=leak.copy()
    for k in range(3):
        a=orw._sl(3,k,slice(0,-1)); b=orw._sl(3,k,slice(1,None))
        lk[a]+=W[k][a]*(~m[b]); lk[b]+=W[k][a]*(~m[a])
    lk=lk*m; Wc=[]
    for k in range(3):
        mm=np.zeros(W[k].shape); sl=[slice(None)]*3; sl[k]=slice(1,None,2); sl=tuple(sl)
        a=orw._sl(3,k,slice(0,-1)); b=orw._sl(3,k,slice(1,None))
        both=np.zeros(W[k].shape,bool); both[a]=m[a]&m[b]
        mm[sl]=(W[k]*both)[sl]; Wc.append(agg(mm,sh))
    lkc=agg(lk,sh); return Wc,lkc,lkc+faces(Wc),m
levels_=[(W,leak0,dg0,None)]
while np.prod(levels_[-1][1].shape)>64:
    Wc,lk,dg,m=coarsen(*levels_[-1][:3]); levels_[-1]=levels_[-1][:3]+(m,); levels_.append((Wc,lk,dg,None))
om=0.8
def P_(x,sh):
    y=x.repeat(2,0).repeat(2,1).repeat(2,2); return y[:sh[0],:sh[1],:sh[2]]
def vcycle(c,b):
    W_,lk,dg,m=levels_[c]; dinv=np.where(dg>0,1/np.where(dg>0,dg,1),0)
    if c==len(levels_)-1:
        x=om*dinv*b
        for _ in range(7): x=x+om*dinv*(b-Aop(W_,dg,x))
        return x
    x=om*dinv*b; res=b-Aop(W_,dg,x)
    xc=vcycle(c+1,agg(res*m,levels_[c+1][1].shape))
    x=x+P_(xc,b.shape)*m
    return x+om*dinv*(b-Aop(W_,dg,x))
def pcg(prec,tol,dt=np.float64,maxit=20000):
    b=np.where(unk,S.rhs*s,0).astype(dt); bb=float((b.astype(float)**2).sum())
    y=np.zeros(shape3,dt); r=b.copy(); z=prec(r).astype(dt); p=z.copy(); rz=float((r*z).sum()); it=0
    Wd=[w.astype(dt) for w in W]; dgd=dg0.astype(dt)
    while float((r.astype(float)**2).sum())>tol*tol*bb and it<maxit:
        q=Aop(Wd,dgd,p).astype(dt); al=rz/float((p*q).sum()); y=(y+dt(al)*p).astype(dt); r=(r-dt(al)*q).astype(dt)
        z=prec(r.astype(float)).astype(dt); rzn=float((r*z).sum()); p=(z+dt(rzn/rz)*p).astype(dt); rz=rzn; it+=1
    x=y.astype(float)*s; prob=np.where(unk,x,S.dvals)
    return prob.reshape(ref.shape),it
for dt in (np.float64,np.float32):
  for nm,pr in [("jacobi",lambda r: r*unk),("mg",lambda r: vcycle(0,r))]:
    prob,it=pcg(pr,1e-7,dt)
    print(dt.__name__,nm,"iters",it,"err",np.abs(prob-ref).max())
