import numpy as np
np.show_config(mode='dicts') if False else None
from threadpoolctl import threadpool_info
print([ (i['internal_api'], i.get('architecture'), i.get('version')) for i in threadpool_info()])
rng=np.random.default_rng(0)
f32=np.float32
def fma(a,b,c):  # exact fma in float32 via float64 (products exact in f64; sum rounding once)
    return f32(np.float64(a)*np.float64(b)+np.float64(c))
def seq_fma(r,x):
    s=f32(0)
    for k in range(len(x)): s=fma(r[k],x[k],s)
    return s
def seq_mul(r,x):
    s=f32(0)
    for k in range(len(x)): s=f32(s+f32(r[k]*x[k]))
    return s
def lanes(r,x,W,tree):
    acc=[f32(0)]*W
    for k in range(len(x)):
        acc[k%W]=fma(r[k],x[k],acc[k%W])
    return tree(acc)
def tree_pairwise(a):
    a=list(a)
    while len(a)>1:
        h=len(a)//2
        a=[f32(a[i]+a[i+h]) for i in range(h)]
    return a[0]
def tree_seq(a):
    s=a[0]
    for v in a[1:]: s=f32(s+v)
    return s
