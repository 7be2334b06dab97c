"""Convergence history of cyclic one-sided Jacobi (circle ordering, the rotation test and absolute floor of
the library kernels) in numpy: the largest relative coupling eta of every sweep, for random / graded / low-rank
R factors.  Supports the early exit of the packed and block Jacobi kernels (jacobi_kpred in csrc/k_small.cu):
each working sweep's eta is about the square of the previous one.  Usage: jacobi_conv_sim.py [SEED]"""
import numpy as np, sys
def run(R, tol):
    X = R.T.copy(); n = X.shape[1]; P = n + (n % 2)
    hist = []
    for sweep in range(30):
        nrm = (X*X).sum(0); mx = nrm.max(); floor = 1e-2*2**-52*mx
        etamax = 0.0; rot = False
        for r in range(P-1):
            for pi in range(P//2):
                if pi == 0: a, b = r, P-1
                else: a = (r+pi) % (P-1); b = (r-pi) % (P-1)
                if a >= n or b >= n: continue
                p, q = min(a,b), max(a,b)
                al, be, ga = X[:,p]@X[:,p], X[:,q]@X[:,q], X[:,p]@X[:,q]
                if ga*ga > tol*tol*al*be and abs(ga) > floor:
                    etamax = max(etamax, abs(ga)/np.sqrt(al*be)); rot = True
                    zeta = (be-al)/(2*ga); t = np.sign(zeta)/(abs(zeta)+np.sqrt(1+zeta*zeta)) if zeta != 0 else 1.0
                    c = 1/np.sqrt(1+t*t); s = c*t
                    xp, xq = X[:,p].copy(), X[:,q].copy()
                    X[:,p] = c*xp - s*xq; X[:,q] = s*xp + c*xq
        hist.append(etamax)
        if not rot: break
    return hist
rng = np.random.default_rng(int(sys.argv[1]) if len(sys.argv)>1 else 0)
for n, kind in [(50,'randn'),(50,'graded'),(64,'randn'),(50,'lowrank')]:
    tol = max(1e-15, n*2**-53)
    if kind == 'randn': B = rng.standard_normal((400, n))
    elif kind == 'graded': B = rng.standard_normal((400, n)) * np.logspace(0, -6, n)
    else: B = rng.standard_normal((400, 40)) @ rng.standard_normal((40, n)) + 1e-3*rng.standard_normal((400,n))
    R = np.linalg.qr(B, mode='r')
    h = run(R, tol)
    print(n, kind, len(h), ' '.join(f'{x:.1e}' for x in h), 'tol', f'{tol:.1e}')
