"""Offline bank-conflict model of the slab-staged K2 LDS pattern (vectorized):
for sampled (view, tile) CTAs of c4 / c5, emulate the warp's lockstep pair
loop per slab and count shared-memory wavefronts per LDS for box layouts."""
import math, sys
import numpy as np

def geom(cfg):
    if cfg == 'c4':
        return 512, 0.5, 1248, 960, 0.64, 496, 220*math.pi/180
    return 1024, 0.25, 2048, 1536, 0.4, 720, 2*math.pi

def rays(cfg, view, u0, v0, TU, TV):
    n, sp, nu, nv, du, nviews, rng = geom(cfg)
    sid, sdd = 750.0, 1200.0
    th = view * rng / nviews
    c, s = math.cos(th), math.sin(th)
    src = np.array([-sid * c, -sid * s, 0.0])
    iu = u0 + np.arange(TU); iv = v0 + np.arange(TV)
    U = (iu - (nu - 1) / 2) * du; V = (iv - (nv - 1) / 2) * du
    UU, VV = np.meshgrid(U, V)
    d = np.stack([sdd * c - UU * s, sdd * s + UU * c, VV], -1)
    d /= np.linalg.norm(d, axis=-1, keepdims=True)
    org = -(n - 1) / 2 * sp
    lo, hi = org - sp, org + n * sp
    t0 = np.full(d.shape[:2], -1e300); t1 = np.full(d.shape[:2], 1e300)
    for ax in range(3):
        with np.errstate(divide='ignore', invalid='ignore'):
            ta = (lo - src[ax]) / d[..., ax]; tb = (hi - src[ax]) / d[..., ax]
        t0 = np.maximum(t0, np.minimum(ta, tb)); t1 = np.minimum(t1, np.maximum(ta, tb))
    hit = t1 > t0
    step = 0.5 * sp
    ns = np.where(hit, np.ceil((t1 - t0) / step), 0).astype(int)
    dt = np.where(hit, (t1 - t0) / np.maximum(ns, 1), 0)
    return (src - org) / sp, d / sp, t0, dt, ns, hit

def wavefronts(addr, valid):
    # addr [R, 32] int, valid [R, 32] -> wavefronts per row
    A = np.where(valid, addr, -1)
    A = np.sort(A, 1)
    dup = np.zeros_like(A, bool); dup[:, 1:] = A[:, 1:] == A[:, :-1]
    keep = (A >= 0) & ~dup
    bank = np.where(keep, A % 32, 32)
    cnt = (bank[..., None] == np.arange(32)).sum(1)
    return cnt.max(1)

def schedule(cell, N, hh, dax, T):
    """lockstep pair loop per slab: list of [32] sample indices (-1 idle)"""
    dcell = cell[..., dax]
    kmax = cell.shape[1]
    valid = (np.arange(kmax)[None] < N[:, None]) & hh[:, None]
    dv = dcell[valid]
    sgn = 1 if np.mean(np.diff(dcell[hh][0][:max(2, N[hh][0])])) >= 0 else -1
    cmin, cmax = dv.min() - 1, dv.max() + 1
    nsl = (cmax - cmin + T) // T
    kk = np.zeros(32, int)
    its = []; d0s = []
    for i in range(nsl):
        s0 = cmin + i * T if sgn > 0 else cmax + 1 - (i + 1) * T
        d0 = s0 if sgn > 0 else s0 - 1
        ends = kk.copy()
        for l in range(32):
            if not hh[l]: continue
            row = dcell[l, :N[l]]
            if sgn > 0: e = np.searchsorted(row, s0 + T - 1, side='right')
            else: e = np.searchsorted(-row, -s0, side='right')
            ends[l] = max(kk[l], e)
        pairs = (ends - kk + 1) // 2
        for p in range(pairs.max() if len(pairs) else 0):
            for half in (0, 1):
                k = kk + 2 * p + half
                ok = (p < pairs) & (k < N) & hh
                its.append(np.where(ok, k, -1)); d0s.append(d0)
        kk = np.minimum(kk + 2 * pairs, N)
    return its, d0s

def sim(cfg, view, u0, v0, layouts, warp=(8, 4), T=8, tile=(16, 16)):
    TU, TV = tile
    o, e, t0, dt, ns, hit = rays(cfg, view, u0, v0, TU, TV)
    if hit.sum() == 0: return None
    es = e[hit].sum(0)
    dax = 0 if abs(es[0]) > abs(es[1]) else 1
    hax = 1 - dax
    wu, wv = warp
    res = {L: [0, 0] for L in layouts}
    for wy in range(TV // wv):
        for wx in range(TU // wu):
            sl = (slice(wy * wv, (wy + 1) * wv), slice(wx * wu, (wx + 1) * wu))
            hh = hit[sl].ravel()
            if hh.sum() == 0: continue
            N = ns[sl].ravel(); kmax = N.max()
            k = np.arange(kmax)
            t = t0[sl].ravel()[:, None] + (k[None] + 0.5) * dt[sl].ravel()[:, None]
            P = o[None, None] + t[..., None] * e[sl].reshape(-1, 3)[:, None]
            cell = np.floor(P).astype(np.int64)
            its, d0s = schedule(cell, N, hh, dax, T)
            if not its: continue
            K = np.array(its); D0 = np.array(d0s)[:, None]
            val = K >= 0
            C = cell[np.arange(32)[None], np.maximum(K, 0)]  # [R, 32, 3]
            for (WH, HZ) in layouts:
                tot = 0
                for dh in (0, 1):
                    for dz in (0, 1):
                        for dd in (0, 1):
                            addr = (C[..., hax] + dh) + WH * (C[..., 2] + dz) + WH * HZ * (C[..., dax] + dd - D0)
                            tot += wavefronts(addr, val).sum()
                res[(WH, HZ)][0] += tot; res[(WH, HZ)][1] += 8 * len(its)
    return res

if __name__ == '__main__':
    cfg = sys.argv[1]
    warp = tuple(int(x) for x in sys.argv[2].split('x')) if len(sys.argv) > 2 else (8, 4)
    tile = tuple(int(x) for x in sys.argv[3].split('x')) if len(sys.argv) > 3 else (16, 16)
    ncase = int(sys.argv[4]) if len(sys.argv) > 4 else 60
    rs = np.random.RandomState(1)
    n, sp, nu, nv, du, nviews, rng = geom(cfg)
    cases = [(int(rs.randint(nviews)), int(rs.randint(nu // tile[0])) * tile[0],
              int(rs.randint(nv // tile[1])) * tile[1]) for _ in range(ncase)]
    layouts = [(40, 24), (44, 24), (36, 24), (48, 24), (52, 24), (56, 24), (72, 24), (68, 24),
               (32, 24), (40, 12), (44, 12), (48, 12), (52, 12), (36, 12)]
    tot = {L: [0, 0] for L in layouts}
    for v, u0, v0 in cases:
        r = sim(cfg, v, u0, v0, layouts, warp, tile=tile)
        if r:
            for L in layouts: tot[L][0] += r[L][0]; tot[L][1] += r[L][1]
    for L in layouts:
        print(cfg, warp, L, 'wf/ld %.3f' % (tot[L][0] / max(tot[L][1], 1)), flush=True)
