"""Pure-Python emulation of the K2 index build + K1 lookup of csrc/index.cu, compared with
the brute-force oracle lookup on random pools (a development aid used to debug the GPU
algorithm on CPU; neither side imports it).  Usage: python scripts/index_emulator.py V Lmin M k
"""
import numpy as np, sys
sys.path.insert(0,'/root/repo')
import oracle as orc
B=0x9E3779B97F4A7C15; MASK=(1<<64)-1
def H(w):
    h=0
    for t in w: h=(h*B+(t+1))&MASK
    return h
def build(seqs, sp, M, K):
    T=[]; ss=[]; se=[]; po=[]
    for s,P in zip(seqs,sp):
        a=len(T); T+=list(s); b=len(T)
        for i in range(a,b): ss.append(a); se.append(b); po.append(P)
    n=len(T); D=M+K
    fu=[10**9]*n; runid_pos=[0]*n
    act=list(range(n)); levels=[]
    for l in range(1,D+1):
        if not act: break
        keys=[((po[i] if l==1 else runid_pos[i]), T[i+l-1]) for i in act]
        order=sorted(range(len(act)), key=lambda a: keys[a])
        pos_sorted=[act[a] for a in order]; ks=[keys[a] for a in order]
        runstart=[]; parent=[]; rid=[]
        for r in range(len(ks)):
            if r==0 or ks[r]!=ks[r-1]:
                runstart.append(r); parent.append(ks[r][0] if l>1 else -1)
            rid.append(len(runstart)-1)
        runstart.append(len(ks))
        nxt=[]
        for r,i in enumerate(pos_sorted):
            R=rid[r]; size=runstart[R+1]-runstart[R]; runid_pos[i]=R
            if size==1: fu[i]=l
            elif i+l<se[i]: nxt.append(i)
        levels.append((pos_sorted,runstart,parent))
        act=nxt
    table={}
    for i in range(n):
        if fu[i] > M: continue
        hi = min(M, se[i]-i)
        if i+1 < se[i]: hi = min(hi, fu[i+1])
        for l2 in range(fu[i], hi+1):
            q=min(K,se[i]-(i+l2))
            table[(po[i],l2,H(T[i:i+l2]))]=(i,q,True,q>0)
    L=len(levels); pq_child=None; po_child=None
    for li in range(L-1,-1,-1):
        l=li+1; pos_sorted,runstart,parent=levels[li]; nr=len(runstart)-1
        top = li==L-1
        if not top:
            cps,crs,cpar=levels[li+1]; cbeg={}; cend={}
            for C in range(len(crs)-1):
                p=cpar[C]
                if C==0 or cpar[C-1]!=p: cbeg[p]=C
                if C==len(crs)-2 or cpar[C+1]!=p: cend[p]=C+1
        pq=[0]*nr; poc=[0]*nr
        for R in range(nr):
            rs=runstart[R]; size=runstart[R+1]-rs; i0=pos_sorted[rs]
            if size==1:
                continue
            q=0; occ=i0
            if not top:
                best=-1;bsz=0
                for C in range(cbeg.get(R,0),cend.get(R,0)):
                    sz=crs[C+1]-crs[C]
                    if sz>bsz: bsz=sz;best=C
                if best>=0:
                    cpos=cps[crs[best]]
                    if bsz==1: occ=cpos; q=min(K,se[cpos]-cpos-l)
                    else: q=min(K,1+pq_child[best]); occ=po_child[best]
            pq[R]=q; poc[R]=occ
            if l<=M: table[(po[occ],l,H(T[occ:occ+l]))]=(occ,q,False,q>0)
        pq_child,po_child=pq,poc
    return T,ss,table
def lookup(T,ss,table,ctx,P,M,Lmin,k):
    L=len(ctx); mmax=min(M,L)
    found={}
    for m in range(1,mmax+1):
        e=table.get((P,m,H(ctx[L-m:])))
        if e: found[m]=e
    hit=set(found)
    while hit:
        m0=max(hit); occ0,q0,u0,c0=found[m0]
        if T[occ0:occ0+m0]!=ctx[L-m0:]: hit.discard(m0); continue
        if u0 and c0:
            ext=0
            while m0+ext<mmax and occ0-1-ext>=ss[occ0] and T[occ0-1-ext]==ctx[L-m0-1-ext]: ext+=1
            ms=m0+ext; d=T[occ0+m0:occ0+m0+q0]
            break
        cands=[m for m in hit if found[m][3] and (m<m0 if u0 else m<=m0)]
        if not cands: ms=0; d=[]; break
        ms=max(cands); occ,q,u,c=found[ms]
        d=T[occ+ms:occ+ms+q]; break
    else:
        ms=0; d=[]
    if ms<Lmin: ms=0; d=[]
    return d[:k], ms
rng=np.random.default_rng(3*100+8)
import itertools
vocab,Lmin,M,k=int(sys.argv[1]),int(sys.argv[2]),int(sys.argv[3]),int(sys.argv[4])
bad=0
for trial in range(30):
    seqs=[];sp=[]
    for P in range(6):
        for _ in range(int(rng.integers(0,6))):
            seqs.append([int(x) for x in rng.integers(0,vocab,int(rng.integers(0,40)))]); sp.append(P)
    T,ss,table=build(seqs,sp,M,k)
    pools={}
    for s,P in zip(seqs,sp): pools.setdefault(P,[]).append(s)
    for _ in range(100):
        P=int(rng.integers(0,6)); c=[int(x) for x in rng.integers(0,vocab,int(rng.integers(1,40)))]
        want=orc.lookup(pools.get(P,[]),c[-M:],M,Lmin,k)
        got=lookup(T,ss,table,c[-M:],P,M,Lmin,k)
        if list(got[0])!=want[0] or got[1]!=want[1]:
            bad+=1
            if bad<4: print("MISMATCH",c[-M:],P,want,got)
print("bad",bad)
