"""NumPy restatement of the reference hot path (TEST INFRASTRUCTURE ONLY).

An independent CPU restatement of the dual-domain CSC algorithm of
/root/reference/proj (FP64, full complex spectra exactly as the reference
forms them). Only tests/ may import it; it is a checker, never the product.
Pinned against the compiled reference (oracle/_ref) in tests/test_oracle_pins.py.
Every function cites the reference lines it restates.
"""
from __future__ import annotations

import numpy as np

ADMM_REL_TOL = 1e-4       # coding.hpp:41
FILTER_NORM_TOL = 1e-3    # learning.cpp:14


def fwd(x):
    """forward_dft (spectral.cpp:59-68): unnormalised, sign -1, last axes."""
    return np.fft.fft2(x)


def inv(s):
    """inverse_dft (spectral.cpp:76-98): 1/D scaled, real part kept."""
    return np.fft.ifft2(s).real


def pad(d, grid):
    """pad_filter (spectral.cpp:106-122): corner placement; d is (..., mh, mw)."""
    out = np.zeros(d.shape[:-2] + tuple(grid))
    out[..., : d.shape[-2], : d.shape[-1]] = d
    return out


def solve_coding(x, d, beta, rho, max_admm, theta=None, z=None):
    """solve_coding / admm_coding (coding.cpp:166-329, 333-356) for one image."""
    K = d.shape[0]
    grid = x.shape
    dh = fwd(pad(d, grid))                              # :59-61
    sigma = (np.abs(dh) ** 2).sum(0) + 1.0 / rho        # :15-21
    xh = fwd(x)                                         # :69
    theta = np.zeros((K,) + grid) if theta is None else theta.copy()
    z = np.zeros((K,) + grid) if z is None else z.copy()
    stats = dict(admm_iters=0, converged=False, degenerate_dictionary=False, dual_rescaled=False)
    if not np.any(d):                                   # :181-191
        stats.update(converged=True, degenerate_dictionary=True)
        lam = -x
        stats["dual_objective"] = -0.5 * (lam * lam).sum() - (lam * x).sum()
        return np.zeros_like(z), np.zeros_like(theta), lam, stats
    th_h, z_h = fwd(theta), fwd(z)                      # :216-220
    inv_rho = 1.0 / rho
    t_inf = 0.0
    for it in range(1, max_admm + 1):
        w_h = th_h + z_h * inv_rho                      # :224-227
        lam_h = ((dh * w_h).sum(0) - xh * inv_rho) / sigma   # :25-37
        t = inv(np.conj(dh) * lam_h)                    # :77-86, 234
        th_new = np.clip(t - z * inv_rho, -beta, beta)  # :237-238
        dth = th_new - theta
        dz = rho * (th_new - t)
        theta = th_new
        z = z + dz                                      # :243-244
        tt = ((th_new - t) ** 2).sum(); th2 = (th_new ** 2).sum(); t2 = (t ** 2).sum()
        dz2 = (dz ** 2).sum(); z2 = (z ** 2).sum(); dth2 = (dth ** 2).sum()
        t_inf = np.abs(t).max()
        th_h, z_h = fwd(theta), fwd(z)                  # :260-261
        primal = np.sqrt(tt) / max(np.sqrt(th2), np.sqrt(t2), 1.0)   # :264-272
        zc = np.sqrt(dz2) / max(np.sqrt(z2), 1.0)
        thc = np.sqrt(dth2) / max(np.sqrt(th2), 1.0)
        stats.update(admm_iters=it, primal_residual=primal, z_change=zc, theta_change=thc)
        if primal <= ADMM_REL_TOL and zc <= ADMM_REL_TOL and thc <= ADMM_REL_TOL:
            stats["converged"] = True
            break
    lam = inv(lam_h)                                    # :287-291
    stats["dual_infeasibility"] = max(0.0, t_inf - beta)
    if t_inf > beta:                                    # :293-300
        lam = lam * (beta / t_inf)
        stats["dual_rescaled"] = True
    stats["dual_objective"] = -0.5 * (lam * lam).sum() - (lam * x).sum()   # :303-309
    return z, theta, lam, stats


def solve_coding_tcsc(x, d, beta, rho, max_admm, theta=None, z=None):
    """solve_coding_tcsc (tcsc.cpp:211-230): admm_coding (coding.cpp:166-329)
    with the BlockKernel of tcsc.cpp:121-171 for a J-channel signal x (J,H,W)
    and dictionary d (K,J,mh,mw). lambda_hat(w) solves the per-bin J x J
    system (D D^H + I/rho) lambda_hat = sum_k d_hat_jk w_hat_k - x_hat/rho
    (tcsc.cpp:31-88; Woodbury is the same solution); t_hat_k =
    sum_j conj(d_hat_jk) lambda_hat_j (tcsc.cpp:90-102)."""
    K, J = d.shape[:2]
    grid = x.shape[1:]
    dh = fwd(pad(d, grid))                              # (K, J, H, W), tcsc.cpp:195-209
    Dw = np.moveaxis(dh, (0, 1), (-1, -2))              # (H, W, J, K): block(bin)
    G = Dw @ np.conj(np.swapaxes(Dw, -1, -2)) + np.eye(J) / rho   # tcsc.cpp:44-47
    xh = fwd(x)                                         # (J, H, W)
    theta = np.zeros((K,) + grid) if theta is None else theta.copy()
    z = np.zeros((K,) + grid) if z is None else z.copy()
    stats = dict(admm_iters=0, converged=False, degenerate_dictionary=False, dual_rescaled=False)
    if not np.any(d):                                   # coding.cpp:181-191
        stats.update(converged=True, degenerate_dictionary=True)
        lam = -x
        stats["dual_objective"] = -0.5 * (lam * lam).sum() - (lam * x).sum()
        return np.zeros_like(z), np.zeros_like(theta), lam, stats
    th_h, z_h = fwd(theta), fwd(z)
    inv_rho = 1.0 / rho
    t_inf = 0.0
    for it in range(1, max_admm + 1):
        w_h = th_h + z_h * inv_rho
        r = np.einsum("kjhw,khw->hwj", dh, w_h) - np.moveaxis(xh, 0, -1) * inv_rho   # tcsc.cpp:75-80
        lam_h = np.moveaxis(np.linalg.solve(G, r[..., None])[..., 0], -1, 0)         # (J, H, W)
        t = inv(np.einsum("kjhw,jhw->khw", np.conj(dh), lam_h))                     # tcsc.cpp:90-102
        th_new = np.clip(t - z * inv_rho, -beta, beta)
        dth = th_new - theta
        dz = rho * (th_new - t)
        theta = th_new
        z = z + dz
        tt = ((th_new - t) ** 2).sum(); th2 = (th_new ** 2).sum(); t2 = (t ** 2).sum()
        dz2 = (dz ** 2).sum(); z2 = (z ** 2).sum(); dth2 = (dth ** 2).sum()
        t_inf = np.abs(t).max()
        th_h, z_h = fwd(theta), fwd(z)
        primal = np.sqrt(tt) / max(np.sqrt(th2), np.sqrt(t2), 1.0)
        zc = np.sqrt(dz2) / max(np.sqrt(z2), 1.0)
        thc = np.sqrt(dth2) / max(np.sqrt(th2), 1.0)
        stats.update(admm_iters=it, primal_residual=primal, z_change=zc, theta_change=thc)
        if primal <= ADMM_REL_TOL and zc <= ADMM_REL_TOL and thc <= ADMM_REL_TOL:
            stats["converged"] = True
            break
    lam = inv(lam_h)
    stats["dual_infeasibility"] = max(0.0, t_inf - beta)
    if t_inf > beta:
        lam = lam * (beta / t_inf)
        stats["dual_rescaled"] = True
    stats["dual_objective"] = -0.5 * (lam * lam).sum() - (lam * x).sum()
    return z, theta, lam, stats


class LearningOperator:
    """LearningOperator (learning.cpp:24-134)."""

    def __init__(self, maps, support, mu_floor):
        self.zh = fwd(maps)                               # [n][k] spectra, :41-48
        self.dead = ~np.any(maps != 0, axis=(0, 2, 3))    # :50-57
        self.mask = np.zeros(maps.shape[2:], dtype=bool)  # :59-64
        self.mask[: support[0], : support[1]] = True
        self.support = support
        self.mu_floor = mu_floor
        self.mu = np.ones(maps.shape[1])

    def set_mu(self, mu):                                 # :66-81
        self.mu = np.maximum(np.asarray(mu, dtype=np.float64), self.mu_floor)
        return bool(np.any(np.asarray(mu) < self.mu_floor))

    def apply(self, v):                                   # :83-122
        vh = fwd(v)
        live = ~self.dead
        c = np.einsum("nkij,nij->kij", np.conj(self.zh), vh)
        sp = inv(c) * self.mask
        ph = fwd(sp)
        w = np.where(live, 0.5 / self.mu, 0.0)
        acc = np.einsum("k,nkij,kij->nij", w, self.zh, ph)
        return v + inv(acc)


def gamma_solve(op, xs, cg_tol, cg_max, gamma):
    """gamma_solve (learning.cpp:136-185), warm started."""
    b = -xs
    bn = np.sqrt((b * b).sum())
    if bn == 0.0:
        return np.zeros_like(gamma), 0, True
    r = b - op.apply(gamma)
    rr = (r * r).sum()
    if np.sqrt(rr) / bn <= cg_tol:
        return gamma, 0, True
    p = r.copy()
    iters, conv = 0, False
    for it in range(1, cg_max + 1):
        ap = op.apply(p)
        pap = (p * ap).sum()
        if pap <= 0.0:
            break
        alpha = rr / pap
        gamma = gamma + alpha * p
        r = r - alpha * ap
        rr_new = (r * r).sum()
        iters = it
        if np.sqrt(rr_new) / bn <= cg_tol:
            conv = True
            break
        p = r + (rr_new / rr) * p
        rr = rr_new
    return gamma, iters, conv


def d_recover(op, gamma, mu):
    """d_recover (learning.cpp:187-216)."""
    gh = fwd(gamma)
    c = np.einsum("nkij,nij->kij", np.conj(op.zh), gh)
    sp = inv(c)[:, : op.support[0], : op.support[1]]
    return sp * (-0.5 / np.maximum(mu, 1e-300))[:, None, None]


def solve_learning(xs, maps, support, cfg, gamma=None, mu=None):
    """solve_learning (learning.cpp:227-355), J = 1."""
    K = maps.shape[1]
    mu = np.ones(K) if mu is None else np.array(mu, dtype=np.float64)
    gamma = np.zeros(xs.shape) if gamma is None else np.array(gamma, dtype=np.float64)
    stats = dict(mu_iters=0, cg_iters=0, converged=False, degenerate=False)
    if not np.any(maps):                                  # :258-270
        stats["degenerate"] = True
        return np.zeros((K,) + tuple(support)), np.zeros_like(gamma), mu, stats
    op = LearningOperator(maps, support, cfg["mu_floor"])
    norms = np.zeros(K)
    d = None
    for it in range(1, cfg["max_mu_iters"] + 1):         # :288-328
        op.set_mu(mu)
        mu = op.mu.copy()
        gamma, cgi, _ = gamma_solve(op, xs, cfg["cg_tol"], cfg["cg_max"], gamma)
        stats["cg_iters"] += cgi
        d = d_recover(op, gamma, mu)
        norms = np.sqrt((d ** 2).sum(axis=(1, 2)))
        stats["mu_iters"] = it
        at_b = np.abs(norms - 1.0) <= FILTER_NORM_TOL
        inact = (mu <= cfg["mu_floor"] * (1.0 + 1e-9)) & (norms < 1.0)
        if np.all(at_b | inact):
            stats["converged"] = True
            break
        if it < cfg["max_mu_iters"]:
            mu = np.maximum(mu * norms, cfg["mu_floor"])     # mu_update :218-225
    scale = np.where(norms > 1.0, 1.0 / np.where(norms > 0, norms, 1.0), 1.0)   # :333-344
    return d * scale[:, None, None], gamma, mu, stats


def objective(x, d, z, beta):
    """evaluate_objective (objective.cpp:59-81), circular convolution via the DFT."""
    rec = inv((fwd(pad(d, x.shape)) * fwd(z)).sum(0))
    r = rec - x
    data = 0.5 * (r * r).sum()
    l1 = beta * np.abs(z).sum()
    return data, l1, data + l1


def init_dictionary(K, support, seed):
    """init_variables (pipeline.cpp:123-156): mt19937_64 uniform [-0.5, 0.5), unit norm."""
    mt = _MT19937_64(seed)
    M = support[0] * support[1]
    d = np.array([[(mt.next() >> 11) * 2.0 ** -53 - 0.5 for _ in range(M)] for _ in range(K)])
    n = np.sqrt((d * d).sum(1))
    d = d / np.where(n == 0, 1.0, n)[:, None]
    return d.reshape(K, support[0], support[1])


class _MT19937_64:
    """std::mt19937_64 (the C++ standard's parameters), for init_variables."""

    def __init__(self, seed):
        self.mt = [0] * 312
        self.mt[0] = seed & 0xFFFFFFFFFFFFFFFF
        for i in range(1, 312):
            self.mt[i] = (6364136223846793005 * (self.mt[i - 1] ^ (self.mt[i - 1] >> 62)) + i) & 0xFFFFFFFFFFFFFFFF
        self.i = 312

    def next(self):
        if self.i >= 312:
            for j in range(312):
                x = (self.mt[j] & 0xFFFFFFFF80000000) | (self.mt[(j + 1) % 312] & 0x7FFFFFFF)
                xa = x >> 1
                if x & 1:
                    xa ^= 0xB5026F5AA96619E9
                self.mt[j] = self.mt[(j + 156) % 312] ^ xa
            self.i = 0
        y = self.mt[self.i]
        self.i += 1
        y ^= (y >> 29) & 0x5555555555555555
        y ^= (y << 17) & 0x71D67FFFEDA60000
        y ^= (y << 37) & 0xFFF7EEE000000000
        y ^= y >> 43
        return y & 0xFFFFFFFFFFFFFFFF


def run_csc(xs, K, support, cfg):
    """run_csc (pipeline.cpp:158-301), normalize = None; returns trace and final state."""
    N = xs.shape[0]
    beta = cfg["beta"]
    d = init_dictionary(K, support, cfg["seed"])
    maps = np.zeros((N, K) + xs.shape[1:])
    theta = np.zeros_like(maps)
    zst = np.zeros_like(maps)
    gamma, mu = None, None
    img = [objective(xs[n], d, maps[n], beta) for n in range(N)]
    prev = sum(o[0] for o in img) + sum(o[1] for o in img)
    trace = []
    for outer in range(1, cfg["max_outer"] + 1):
        admm_total = 0
        zc2 = zn2 = 0.0
        for n in range(N):
            z, th, _, st = solve_coding(xs[n], d, beta, cfg["rho"], cfg["max_admm"], theta[n], zst[n])
            theta[n], zst[n] = th, z
            admm_total += st["admm_iters"]
            cand = objective(xs[n], d, z, beta)
            if cand[2] <= img[n][2]:                       # :236
                zc2 += ((z - maps[n]) ** 2).sum()
                maps[n] = z
                img[n] = cand
            zn2 += (maps[n] ** 2).sum()
        data = sum(o[0] for o in img)
        l1 = sum(o[1] for o in img)
        trace.append(dict(phase=0, total=data + l1, data_term=data, l1_term=l1, admm_iters=admm_total))
        dc, gamma, mu, ls = solve_learning(xs, maps, support, cfg, gamma, mu)
        cand = sum(objective(xs[n], dc, maps[n], beta)[0] for n in range(N))
        dchg = 0.0
        if cand <= data:                                   # :272
            dchg = ((dc - d) ** 2).sum()
            d = dc
            img = [objective(xs[n], d, maps[n], beta) for n in range(N)]
            data = cand
        trace.append(dict(phase=1, total=data + l1, data_term=data, l1_term=l1, cg_iters=ls["cg_iters"],
                          mu_iters=ls["mu_iters"]))
        total = data + l1
        oc = abs(prev - total) / max(abs(prev), 1e-30)
        zc = np.sqrt(zc2) / max(np.sqrt(zn2), 1.0)
        dcg = np.sqrt(dchg) / max(np.sqrt((d * d).sum()), 1.0)
        prev = total
        if oc <= cfg["tol"] and zc <= cfg["tol"] and dcg <= cfg["tol"]:
            break
    return dict(trace=trace, dict=d, maps=maps)
