#!/usr/bin/env python
"""Certificate-policy simulation (design data for DESIGN.md §5.7, not a test):
the per-pass transforms of a real run (tools/dump_T.py JSON) applied to a
sample of the large16m source; a query keeps its k-list certificate while its
displacement since the last search stays below rho = max(L_(k+1) - dmax,
(L_(k+1) - d_1) / 2) (exact distances from a scipy KD-tree; targets outside
the 27-cell stencil bounded by h + the face gap, 2h + gap when the 5^3
neighbourhood is empty). Prints the live re-searches and dead re-checks per
pass for k = 1 and 3.
usage: cert_sim.py T_init.json N   (expects /tmp/l16_src.npy, /tmp/l16_tgt.npy
from synth.make("large16m"))"""
import numpy as np, json, sys
from scipy.spatial import cKDTree
src=np.load('/tmp/l16_src.npy'); tgt=np.load('/tmp/l16_tgt.npy')
Ts=[np.array(t) for t in json.load(open(sys.argv[1]))['T']]
tree=cKDTree(tgt.astype(np.float64))
rng=np.random.default_rng(1); idx=rng.choice(len(src),int(sys.argv[2]),replace=False)
s=src[idx].astype(np.float64)
dmax=0.05; h=dmax*(1+2**-20); o=tgt.min(0).astype(np.float64)
ct=np.floor((tgt.astype(np.float64)-o)/h).astype(np.int64)+2
M=4096
occ=np.unique((ct[:,2]*M+ct[:,1])*M+ct[:,0])
def nonempty(p, r):
    c=np.floor((p-o)/h).astype(np.int64)+2
    res=np.zeros(len(p),bool)
    for dz in range(-r,r+1):
        for dy in range(-r,r+1):
            for dx in range(-r,r+1):
                k=((c[:,2]+dz)*M+c[:,1]+dy)*M+c[:,0]+dx
                j=np.minimum(np.searchsorted(occ,k),len(occ)-1); res|=occ[j]==k
    return res
KMAX=5
def cert(Pk, sel, k):
    p=Pk[sel]
    d,_=tree.query(p,k=KMAX,distance_upper_bound=3*h)
    c=(p-o)/h; f=c-np.floor(c); mfg=np.minimum(f,1-f).min(1)*h
    live=nonempty(p,1)
    reach=h+mfg
    far=~nonempty(p,2)
    reach=np.where(far, reach+h, reach)
    D=np.minimum(d,reach[:,None])
    if k==0: rho=D[:,0]-dmax
    else:
        L=D[:,k]; U=D[:,0]; rho=np.maximum(L-dmax,(L-U)/2)
    rho=np.where(live, rho, reach-dmax)
    return rho, live
for k in (1,3):
    Pb=P=None
    Pb=s@Ts[0][:3,:3].T+Ts[0][:3,3]
    rho,live=cert(Pb,np.ones(len(s),bool),k); base=np.zeros(len(s),int)
    srch=[];dead=[]
    for kk in range(1,len(Ts)):
        Pk=s@Ts[kk][:3,:3].T+Ts[kk][:3,3]; eps=np.linalg.norm(Pk-Pb,axis=1)
        bad=(eps>=rho)|(kk-base>32)
        r2,l2=cert(Pk,bad,k); rho[bad]=r2; Pb[bad]=Pk[bad]; base[bad]=kk
        srch.append(l2.sum()/len(s)); dead.append((~l2).sum()/len(s))
    print('list k',k,'live searches/pass %.3f  dead rechecks/pass %.3f'%(np.mean(srch),np.mean(dead)),' '.join('%.3f'%x for x in srch[:6]),flush=True)
