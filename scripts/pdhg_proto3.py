# SPDX-License-Identifier: Apache-2.0
"""numpy prototype: restarted reflected Halpern PDHG (experiments only)."""
import sys, os, time
import numpy as np
sys.path.insert(0, os.path.dirname(os.path.abspath(__file__)))
from pdhg_proto import model


def solve(K, c, b, sense, lb, ub, tol=1e-6, max_iters=100000, verbose=False, ruiz=10, cap=None, check=64,
          reflect=True):
    if cap is not None:
        c = np.minimum(c, cap)
    m, n = K.shape
    Dr, Dc = np.ones(m), np.ones(n)
    A = abs(K).tocsr()
    for it in range(ruiz + 1):
        S = (A.multiply(Dr[:, None])).multiply(Dc[None, :]).tocsr()
        if it < ruiz:
            rn = np.asarray(S.max(axis=1).todense()).ravel(); cn = np.asarray(S.max(axis=0).todense()).ravel()
        else:
            rn = np.asarray(S.sum(axis=1)).ravel(); cn = np.asarray(S.sum(axis=0)).ravel()
        Dr[rn > 0] /= np.sqrt(rn[rn > 0]); Dc[cn > 0] /= np.sqrt(cn[cn > 0])
    Ks = K.multiply(Dr[:, None]).multiply(Dc[None, :]).tocsr(); KsT = Ks.T.tocsr()
    cs, lbs, ubs, bs = c * Dc, lb / Dc, ub / Dc, b * Dr
    cscale = 1.0 / (np.linalg.norm(cs) + 1.0); bscale = 1.0 / (np.linalg.norm(bs) + 1.0)
    cs, bs, lbs, ubs = cs * cscale, bs * bscale, lbs * bscale, ubs * bscale
    G, L = sense == 'G', sense == 'L'
    v = np.ones(n)
    for _ in range(80):
        v = KsT @ (Ks @ v); lam = np.linalg.norm(v); v /= lam
    eta = 0.998 / np.sqrt(lam)
    bl2 = np.linalg.norm(b)
    def kkt(x, y):
        r = Ks @ x - bs
        viol = np.where(sense == 'E', r, np.where(G, np.minimum(r, 0), np.maximum(r, 0))) / Dr / bscale
        rc = cs - KsT @ y
        pobj = cs @ x / cscale / bscale; dobj = (bs @ y + np.sum(np.where(rc > 0, lbs * rc, ubs * rc))) / cscale / bscale
        gap = abs(pobj - dobj) / (1 + abs(pobj) + abs(dobj)); pres = np.linalg.norm(viol) / (1 + bl2)
        return gap, pres, pobj, dobj
    def werr(x, y, w):
        r = Ks @ x - bs
        pv = np.where(sense == 'E', r, np.where(G, np.minimum(r, 0), np.maximum(r, 0)))
        rc = cs - KsT @ y
        pobj = cs @ x; dobj = bs @ y + np.sum(np.where(rc > 0, lbs * rc, ubs * rc))
        return np.sqrt(w * (pv @ pv) + (pobj - dobj) ** 2 / 1.0)
    w = 1.0
    x = np.zeros(n); y = np.zeros(m); x0, y0 = x.copy(), y.copy()
    k = 0; total = 0; restarts = 0
    last = werr(x, y, w); prev = last
    while total < max_iters:
        tau, sig = eta / w, eta * w
        xt = np.clip(x - tau * (cs - KsT @ y), lbs, ubs)
        yt = y + sig * (bs - Ks @ (2 * xt - x))
        yt[G] = np.maximum(yt[G], 0); yt[L] = np.minimum(yt[L], 0)
        total += 1
        if reflect:
            x = (k + 1) / (k + 2) * (2 * xt - x) + x0 / (k + 2)
            y = (k + 1) / (k + 2) * (2 * yt - y) + y0 / (k + 2)
        else:
            x = (k + 1) / (k + 2) * xt + x0 / (k + 2)
            y = (k + 1) / (k + 2) * yt + y0 / (k + 2)
        k += 1
        if total % check == 0:
            cur = werr(xt, yt, w)
            if verbose and (total // check) % 200 == 0:
                g, p, po, do = kkt(xt, yt)
                print(total, "p=%.10g d=%.10g gap=%.2e pres=%.2e w=%.3g" % (po, do, g, p, w))
            g, p, po, do = kkt(xt, yt)
            if g <= tol and p <= tol:
                return (g, p, po, do), total, restarts
            if cur <= 0.2 * last or (cur <= 0.8 * last and cur > prev) or k >= 0.36 * total:
                ddx, ddy = np.linalg.norm(xt - x0), np.linalg.norm(yt - y0)
                if ddx > 1e-10 and ddy > 1e-10:
                    w = np.exp(0.5 * np.log(ddy / ddx) + 0.5 * np.log(w))
                x, y = xt.copy(), yt.copy(); x0, y0 = x.copy(), y.copy(); k = 0
                last = werr(x, y, w); restarts += 1
            prev = cur
    return kkt(xt, yt), total, restarts
