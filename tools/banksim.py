"""Shared-memory bank-conflict simulation of the forward RMW lane mappings.

Draws random top-k column sets of N(0,1) rows and reports the mean wavefronts (max distinct words per bank)
per 32-lane shared-memory instruction for several lane mappings / buffer layouts."""
import numpy as np
rng=np.random.default_rng(0)
H=256
def rows(n,k):
    x=rng.standard_normal((n,H))
    idx=np.sort(np.argpartition(-x,k-1,axis=1)[:,:k],axis=1)
    return idx
def degree(addr):  # addr: (..., 32) word addresses -> wavefronts = max distinct words per bank
    bank=addr%32
    out=[]
    for a,b in zip(addr.reshape(-1,32),bank.reshape(-1,32)):
        d={}
        for aa,bb in zip(a,b): d.setdefault(bb,set()).add(aa)
        out.append(max(len(s) for s in d.values()))
    return np.mean(out)
def sim(k, V, layout, n=4000, stride_map=False, off=0):
    SW=min(32,k//V); EPI=32//SW
    idx=rows(n*EPI,k).reshape(n,EPI,k)
    res=[]
    for v in range(V):
        # lane (sub b, p) accesses entry e
        if stride_map: ent=np.array([p + SW*v for p in range(SW)])
        else: ent=np.array([p*V+v for p in range(SW)])
        cols=idx[:,:,ent]  # n, EPI, SW
        b=np.arange(EPI)[None,:,None]
        addr=layout(cols)+b*(H+off)
        res.append(degree(addr))
    return np.mean(res)
ident=lambda c:c
swz=lambda c: c ^ (((c>>5)&7)<<2)
swz2=lambda c: (c & ~31) | ((c + 5*(c>>5)) & 31)
for k,V in [(32,4),(32,2),(32,1),(16,2),(8,1),(64,4)]:
    print(k,V,'contig id %.2f'%sim(k,V,ident),'off8 %.2f'%sim(k,V,ident,off=8),'swz %.2f'%sim(k,V,swz),'swz+off %.2f'%sim(k,V,swz,off=8),'rot5 %.2f'%sim(k,V,swz2,off=8), 'stride %.2f'%sim(k,V,ident,stride_map=True),'stride+off8 %.2f'%sim(k,V,ident,stride_map=True,off=8))
