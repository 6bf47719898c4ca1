"""Fit of R(t) = erfcx(t/sqrt2)/2 used by the fp32 GeLU estimate in csrc/zq_rowops.cu
(gelu_est), and an fp32-emulated check of the estimate's relative error."""
import numpy as np
from scipy.special import erfcx, erfc
f32=np.float32
T=5.6
t=np.linspace(0,T,400001)
R=0.5*erfcx(t/np.sqrt(2))
res={}
for deg in [6,7,8]:
  for c in np.linspace(0.2,0.5,31):
    y=1/(1+c*t); w=1/R
    V=np.vander(y,deg+1,increasing=True); wt=np.ones_like(t)
    for it in range(40):
        coef=np.linalg.lstsq(V*(w*wt)[:,None],R*w*wt,rcond=None)[0]
        err=(V@coef-R)/R; wt=wt*(1+(np.abs(err)/np.abs(err).max())**2)
    e=np.abs(err).max()
    if deg not in res or e<res[deg][0]: res[deg]=(e,c,coef)
for deg,(e,c,coef) in res.items(): print(deg,c,e)
deg=6; e,c,coef=res[deg]
cf=coef.astype(f32); c32=f32(c)
# emulate f32 evaluation of gelu_est on dense x
x=np.concatenate([np.linspace(-5.5,10,2000001).astype(f32), (np.random.default_rng(0).standard_normal(2000000)*2).astype(f32)])
x=x[x>=-5.5]
def r32(v): return np.asarray(v,np.float64).astype(f32).astype(np.float64)
tt=np.abs(x).astype(np.float64)
a=r32(tt*tt); err2=tt*tt-a   # fma exact remainder
K=0.5/np.log(2)
khi=float(f32(K)); klo=float(f32(K-khi))
arg=r32(-(a*khi)); arg=r32(arg - (a*klo + err2*khi))  # approx emulation
ex=r32(2.0**arg)*(1+0)      # ex2.approx ~ correctly rounded in emulation
y=r32(1.0/r32(1.0+r32(float(c32)*tt)))
p=np.full_like(y,float(cf[-1]))
for k in range(deg-1,-1,-1): p=r32(p*y+float(cf[k]))
Q=r32(ex*p)
Phi=np.where(x>=0, r32(1.0-Q), Q)
g=r32(x.astype(np.float64)*Phi)
true=0.5*x.astype(np.float64)*erfc(-x.astype(np.float64)/np.sqrt(2))
m=true!=0
rel=np.abs(g[m]-true[m])/np.abs(true[m])
print("max rel err of gelu_est (emulated f32):",rel.max(), "at x=",x[m][rel.argmax()])
print("coefs c=",repr(float(c32)), [repr(float(v)) for v in cf])
