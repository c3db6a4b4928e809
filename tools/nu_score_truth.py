"""The nu component of the score at theta = (1.4305, 0.10122, 1.92930) on the 14 x 14 jittered
grid of tests/test_gpu_likelihood.py::test_oracle_parity_theta_sweep, with dSigma/dnu from
30-digit mpmath values (d/dnu of 2^(1-nu)/Gamma(nu) u^nu K_nu(u)) instead of the reference's
case-2 series: how far the reference (oracle) and the engine are from the truth.  CPU only,
~90 s.  Output recorded in profiles/r02_nu_score_noise.txt."""
import numpy as np, mpmath as mp, sys, time
sys.path.insert(0,'/root/repo')
import importlib.util
from oracle import maternmle_cpu as O
from scipy.spatial.distance import pdist, squareform
from scipy.linalg import cho_factor, cho_solve
mp.mp.dps=30
import paper_2601_11437_b200 as pk
jittered_grid=pk.jittered_grid
rng=np.random.default_rng(41)
loc=jittered_grid(14,5); n=loc.shape[0]; z=rng.standard_normal(n)
th=(1.4304897370021574, 0.10121907877941017, 1.9292950324384652)
s2,a,nu=th
h=pdist(loc); u=h/a
t0=time.time()
# exact dC/dnu = s2 * d/dnu [ 2^(1-nu)/Gamma(nu) * u^nu K_nu(u) ]
def dcdnu(uu):
    uu=mp.mpf(float(uu))
    f=lambda v: mp.power(2,1-v)/mp.gamma(v)*mp.power(uu,v)*mp.besselk(v,uu)
    return float(s2*mp.diff(f, nu))
d=np.array([dcdnu(x) for x in u])
print('mp time',time.time()-t0)
dS=squareform(d)  # zero diagonal (d/dnu of sigma2 = 0)
S=O.matrix(loc, th, 'sigma')
c=cho_factor(S, lower=True)
w=cho_solve(c, z)
W=cho_solve(c, dS)
score_true=0.5*(w@dS@w) - 0.5*np.trace(W)
ll,g,f=O.eval_all(loc,z,th)
print('true-ish score_nu %.9f  oracle %.9f  engine(table) -15643.24268982'%(score_true, g[2]))
dref=O.matrix(loc, th, 'nu') if True else None
print('max rel elementwise err of reference dSigma/dnu vs mpmath: %.2e'%np.max(np.abs(squareform(dref,checks=False)-d)/np.abs(d)))
