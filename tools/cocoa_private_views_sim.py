"""VERDICT r1 next #4 asked for per-CTA private views on C3 (one local pass
per CTA with sigma' = #CTAs, one merge per pass).  This CPU simulation of
exactly that scheme (dual hinge SVM, dense d = 28, lambda scaled with n so
n/lambda matches C3) gives the relative duality gap after each epoch for P
private views: P = 1 is sequential SCD.  Result (profiles/cocoa_private_views_r2.txt):
P = 16 is already ~17x behind after 6 epochs and P = 1024 ~2e4x, so the
HBM-speed epochs of a private-view kernel cannot buy back the epochs.

    python tools/cocoa_private_views_sim.py 220000 2 1,16,64,256,1024 6
"""
import numpy as np, sys, time
n, d, lam = int(sys.argv[1]), 28, float(sys.argv[2])
rng = np.random.default_rng(3)
X = rng.standard_normal((n, d)); X /= np.linalg.norm(X, axis=1, keepdims=True)
w = rng.standard_normal(d)
y = np.where(X @ w + 0.3 * rng.standard_normal(n) >= 0, 1.0, -1.0)
A = X * y[:, None]          # columns a_i (rows of A here)
def gap(alpha):
    v = A.T @ alpha; wv = v / lam
    f = v @ v / (2 * lam); g = -alpha.sum()
    F = f + g
    marg = A @ wv
    # f*(w) + sum g*(-a.w): fconj = lam/2|w|^2 ; g*(s) = max(0, s+1) with s = -a.w
    G = f + lam / 2 * wv @ wv + np.maximum(0, 1 - marg).sum() + g
    return F, G
for P in [int(x) for x in sys.argv[3].split(",")]:
    alpha = np.zeros(n)
    v = np.zeros(d)
    part = np.array_split(np.arange(n), P)
    L = min(len(p) for p in part)
    out = []
    t0 = time.time()
    for ep in range(int(sys.argv[4])):
        # every partition: one local SCD epoch on its first L coords (random order), local view
        idx = np.stack([p[rng.permutation(len(p))[:L]] for p in part])   # P x L
        V = np.tile(v / lam, (P, 1))
        quad = P / lam
        dal = np.zeros(n)
        for t in range(L):
            j = idx[:, t]
            a = A[j]                                    # P x d
            ga = np.einsum("pd,pd->p", a, V)            # view = v/lam + quad*A_k d_k  (scaled below)
            t_ = alpha[j] + dal[j]
            c = quad * 1.0
            tn = np.clip(t_ + (1 - ga) / c, 0, 1)
            st = tn - t_
            dal[j] += st
            V += quad * st[:, None] * a
        # V started at v/lam? fix: view = grad f(v) = v/lam
        alpha += dal
        v = A.T @ alpha
        F, G = gap(alpha)
        out.append(G / abs(F))
    print(P, ["%.2e" % x for x in out], "%.1fs" % (time.time() - t0), flush=True)
