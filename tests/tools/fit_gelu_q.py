"""tests/tools/fit_gelu_q.py -- offline generator (run once; the printed fp32
coefficients are pasted into paper_2210_10246_b200/csrc/gelu_math.h).

Fits P(t) ~ (a + K) * Q(a) * exp(a^2/2), Q(a) = Phi(-a) = erfc(a/sqrt2)/2,
t = (a - K)/(a + K), a in [0, 13], as a polynomial in t with coefficients
rounded to fp32 one at a time (lowest first) and the rest refitted, least
squares in relative error.  Prints (K, degree, max relative fit error,
coefficients highest first).  gelu_math.h uses K = 2.5, degree 10.
"""
import numpy as np, sys
from scipy.special import erfcx
def G(a): return 0.5*erfcx(a/np.sqrt(2))
A=13.0
def fitfloat(K, deg, N=12000):
    tmax=(A-K)/(A+K)
    tt = np.cos(np.pi*(np.arange(N)+0.5)/N)
    tn = -1 + (tt+1)/2*(tmax+1); a = K*(1+tn)/(1-tn); h=(a+K)*G(a)
    fixed=[]
    for k in range(deg+1):
        r = h - np.polynomial.polynomial.polyval(tn, np.array(fixed+[0.0]))
        V = np.stack([tn**j for j in range(k,deg+1)],1)/h[:,None]
        sol,*_ = np.linalg.lstsq(V, r/h, rcond=None)
        fixed.append(float(np.float32(sol[0])))
    ta = np.linspace(-1,tmax,400001); aa=K*(1+ta)/(1-ta)
    e=np.max(np.abs(np.polynomial.polynomial.polyval(ta,np.array(fixed))/((aa+K)*G(aa))-1))
    return fixed, e
for K in [2.0,2.5,3.0]:
  for deg in [9,10,11]:
    f,e=fitfloat(K,deg); print(K,deg,e, ', '.join('%.9ef'%v for v in f[::-1]))
