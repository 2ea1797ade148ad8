# SPDX-License-Identifier: Apache-2.0
"""numpy prototype: PDLP-style PDHG with adaptive steps (experiments only)."""
import sys, os, time
import numpy as np
sys.path.insert(0, os.path.dirname(os.path.abspath(__file__)))
from pdhg_proto import model


def solve(K, c, b, sense, lb, ub, tol=1e-6, max_iters=100000, verbose=False, ruiz=10, cap=None, check=64):
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
    # bound-objective rescaling
    cscale = 1.0 / (np.linalg.norm(cs) + 1.0); bscale = 1.0 / (np.linalg.norm(bs) + 1.0)
    cs, bs, lbs, ubs = cs * cscale, bs * bscale, lbs * bscale, ubs * bscale
    G, L = sense == 'G', sense == 'L'
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
        return np.sqrt(w * w * (pv @ pv) + (pobj - dobj) ** 2)
    x = np.zeros(n); y = np.zeros(m); Kx = Ks @ x
    eta = 1.0 / abs(Ks).max(); w = 1.0
    xs = np.zeros(n); ys = np.zeros(m); wsum = 0.0; xr, yr = x.copy(), y.copy()
    last = werr(x, y, w); prev = last; since = 0; k = 0; restarts = 0; total = 0
    while total < max_iters:
        while True:
            total += 1
            xn = np.clip(x - (eta / w) * (cs - KsT @ y), lbs, ubs)
            Kxn = Ks @ xn
            yn = y + (eta * w) * (bs - (2 * Kxn - Kx))
            yn[G] = np.maximum(yn[G], 0); yn[L] = np.minimum(yn[L], 0)
            dx, dy = xn - x, yn - y
            denom = 2 * abs(dy @ (Kxn - Kx))
            emax = (w * (dx @ dx) + (dy @ dy) / w) / denom if denom > 0 else np.inf
            k += 1
            enew = min((1 - (k + 1) ** -0.3) * emax, (1 + (k + 1) ** -0.6) * eta)
            if eta <= emax:
                x, y, Kx = xn, yn, Kxn
                xs += eta * xn; ys += eta * yn; wsum += eta
                eta = enew
                break
            eta = enew
        since += 1
        if since % check == 0:
            xa, ya = xs / wsum, ys / wsum
            ec, ea = werr(x, y, w), werr(xa, ya, w)
            use_avg = ea < ec; cand = ea if use_avg else ec
            cx, cy = (xa, ya) if use_avg else (x, y)
            g, p, po, do = kkt(cx, cy)
            if verbose and (total // check) % 100 == 0:
                print(total, "p=%.10g d=%.10g gap=%.2e pres=%.2e w=%.3g eta=%.3g" % (po, do, g, p, w, eta))
            if g <= tol and p <= tol:
                return (g, p, po, do), total, restarts
            if cand <= 0.2 * last or (cand <= 0.8 * last and cand > prev) or since >= 0.36 * total:
                x, y = cx.copy(), cy.copy(); Kx = Ks @ x
                ddx, ddy = np.linalg.norm(x - xr), np.linalg.norm(y - yr)
                if ddx > 1e-10 and ddy > 1e-10:
                    w = np.exp(0.5 * np.log(ddy / ddx) + 0.5 * np.log(w))
                xr, yr = x.copy(), y.copy(); xs[:] = 0; ys[:] = 0; wsum = 0.0
                last = werr(x, y, w); since = 0; restarts += 1
            prev = cand
    return kkt(x, y), total, restarts


if __name__ == "__main__":
    sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
    from oracle import xo
    from bench import configs
    name = sys.argv[1]
    doc = configs.fig2_doc() if name == "fig2" else configs.vgg16_doc()
    a = xo.arrays_from_json(doc)
    K, c, b, sense, lb, ub = model(a)
    cap = float(sys.argv[3]) if len(sys.argv) > 3 else None
    t = time.time()
    print(solve(K, c, b, sense, lb, ub, verbose=True, max_iters=int(sys.argv[2]), cap=cap), time.time() - t)
