import numpy as np
exec(open(__file__.replace('blas_order_probe.py', '_order_base.py')).read())
def hreduce_adj(v):
    v=list(v)
    while len(v)>1:
        v=[f32(v[2*i]+v[2*i+1]) for i in range(len(v)//2)]
    return v[0]
def multi(r,x,W,nacc):
    d=len(x); accs=[[f32(0)]*W for _ in range(nacc)]
    for k in range(d):
        blk=k//W; a=accs[blk%nacc]; a[k%W]=fma(r[k],x[k],a[k%W])
    t=accs[0]
    for a in accs[1:]: t=[f32(t[i]+a[i]) for i in range(len(t))]
    return hreduce_adj(t)
for d in (1,2,3,4,5,7,8,9,12,15,16,17,24,31,32,33,48,64,65,96,128):
    A=rng.standard_normal((300,d)).astype(f32); q=rng.standard_normal(d).astype(f32)
    ref=A@q
    out=[]
    for W in (1,2,4,8,16):
        for nacc in (1,2,4):
            got=np.array([multi(A[i],q,W,nacc) for i in range(100)],dtype=f32)
            m=(got==ref[:100]).mean()
            if m>0.97: out.append(f"W{W}n{nacc}")
    print(d,out)
