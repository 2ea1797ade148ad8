# SPDX-License-Identifier: Apache-2.0
"""numpy prototype of the K3 PDHG (same algorithm as csrc/pdhg.cu) for
convergence experiments on the CPU.  Not used by the product."""
import sys, os, time
import numpy as np
from scipy.sparse import csr_matrix
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from oracle import xo
from bench import configs


def model(a, strict=False):
    m = xo.Oracle().build_model(a, strict)
    K = csr_matrix((m.val, m.col, m.row_ptr), shape=(m.n_rows, m.n_cols))
    T, D, E = a.T, a.D, a.E
    FE = E + T
    firstU = 3 * D * T * T + D * T * FE
    ub = np.ones(m.n_cols); ub[m.fixed.astype(bool)] = 0
    for d in range(D):
        ub[firstU + d * T * T: firstU + (d + 1) * T * T] = a.budget[d]
    return K, m.obj.copy(), m.rhs.copy(), m.sense.view('S1').astype(str), np.zeros(m.n_cols), ub


def solve(K, c, b, sense, lb, ub, tol=1e-6, max_iters=200000, block=64, verbose=False, ruiz=10, pc=True,
          omega_mode="norm", adaptive=False, update_w=True, w0=None):
    m, n = K.shape
    Dr, Dc = np.ones(m), np.ones(n)
    A = abs(K).tocsr()
    for it in range(ruiz + (1 if pc else 0)):
        S = (A.multiply(Dr[:, None])).multiply(Dc[None, :]).tocsr()
        if it < ruiz:
            rn = np.asarray(S.max(axis=1).todense()).ravel(); cn = np.asarray(S.max(axis=0).todense()).ravel()
        else:
            rn = np.asarray(S.sum(axis=1)).ravel(); cn = np.asarray(S.sum(axis=0)).ravel()
        Dr[rn > 0] /= np.sqrt(rn[rn > 0]); Dc[cn > 0] /= np.sqrt(cn[cn > 0])
    Ks = K.multiply(Dr[:, None]).multiply(Dc[None, :]).tocsr()
    KsT = Ks.T.tocsr()
    cs, lbs, ubs, bs = c * Dc, lb / Dc, ub / Dc, b * Dr
    # ||Ks||
    v = np.ones(n)
    for _ in range(60):
        v = KsT @ (Ks @ v); lam = np.linalg.norm(v); v /= lam
    eta = 0.95 / np.sqrt(lam)
    omega = np.linalg.norm(cs) / np.linalg.norm(bs) if omega_mode == "norm" else 1.0
    if w0 is not None: omega = w0
    bl2 = np.linalg.norm(b)
    def kkt(x, y):
        Kx = Ks @ x; r = Kx - bs
        viol = np.where(sense == 'E', r, np.where(sense == 'G', np.minimum(r, 0), np.maximum(r, 0))) / Dr
        rc = cs - KsT @ y
        pobj = cs @ x; dobj = bs @ y + np.sum(np.where(rc > 0, lbs * rc, ubs * rc))
        gap = abs(pobj - dobj) / (1 + abs(pobj) + abs(dobj)); pres = np.linalg.norm(viol) / (1 + bl2)
        return gap, pres, pobj, dobj, np.hypot(gap, pres)
    x = np.zeros(n); y = np.zeros(m); xs = np.zeros(n); ys = np.zeros(m); xr = x.copy(); yr = y.copy()
    last = kkt(x, y); prev = last; since = 0; iters = 0; restarts = 0
    G, L = sense == 'G', sense == 'L'
    while iters < max_iters:
        tau, sig = eta / omega, eta * omega
        for _ in range(block):
            xn = np.clip(x - tau * (cs - KsT @ y), lbs, ubs)
            xb = 2 * xn - x; x = xn; xs += xn
            yn = y + sig * (bs - Ks @ xb)
            yn[G] = np.maximum(yn[G], 0); yn[L] = np.minimum(yn[L], 0)
            y = yn; ys += yn
        iters += block; since += block
        cur = kkt(x, y); xa, ya = xs / since, ys / since; av = kkt(xa, ya)
        use_avg = av[4] < cur[4]; cand = av if use_avg else cur
        if verbose and iters % (block * 50) == 0:
            print(iters, "p=%.10g d=%.10g gap=%.2e pres=%.2e w=%.3g" % (cur[2], cur[3], cur[0], cur[1], omega))
        if cand[0] <= tol and cand[1] <= tol:
            return cand, iters, restarts
        if cand[4] <= 0.2 * last[4] or (cand[4] <= 0.8 * last[4] and cand[4] > prev[4]) or since >= 0.36 * iters:
            if use_avg: x, y = xa.copy(), ya.copy()
            dx, dy = np.linalg.norm(x - xr), np.linalg.norm(y - yr)
            if dx > 1e-10 and dy > 1e-10 and update_w: omega = np.exp(0.5 * np.log(dy / dx) + 0.5 * np.log(omega))
            xr, yr = x.copy(), y.copy(); xs[:] = 0; ys[:] = 0; last = cand; since = 0; restarts += 1
        prev = cand
    return cur, iters, restarts


if __name__ == "__main__":
    name = sys.argv[1] if len(sys.argv) > 1 else "fig2"
    doc = configs.fig2_doc() if name == "fig2" else configs.vgg16_doc()
    a = xo.arrays_from_json(doc)
    K, c, b, sense, lb, ub = model(a)
    t = time.time()
    print(solve(K, c, b, sense, lb, ub, verbose=True, max_iters=int(sys.argv[2]) if len(sys.argv) > 2 else 20000), time.time() - t)
