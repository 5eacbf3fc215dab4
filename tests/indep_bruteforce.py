"""Independent brute-force checker for tiny instances (pure Python, test-only).

It pins the oracle's brute-force spaces and closed forms WITHOUT using them:
device frequencies are found by numeric bisection on the latency constraints
(not by D20's closed form), edge time is the sum of per-layer latencies
L_n(f_e, b) = d_n(b) A_n / f_e (Eq. (5)), and the general-vector schedule
is checked by simulating the edge GPU as-soon-as-possible with the candidate
device frequencies (Fig. 1 caption P:75; constraint kinds P:179), rather than by
the oracle's ALAP budget formula.  Results agree with the oracle up to the
bisection tolerance, so comparisons use a relative tolerance.
"""
from __future__ import annotations

import itertools


def _d(model, n, b):
    return float(model.d[n * (model.B_max + 1) + b])


def _c(model, n, b):
    return float(model.c[n * (model.B_max + 1) + b])


def _inst(batch, i):
    o0, o1 = int(batch.user_off[i]), int(batch.user_off[i + 1])
    users = [dict(zeta=batch.zeta[u], kappa=batch.kappa[u], f_min=batch.f_min[u], f_max=batch.f_max[u],
                  R=batch.R[u], p_u=batch.p_u[u], T=batch.T[u]) for u in range(o0, o1)]
    return batch.models[batch.model_id[i]], users, dict(t_free=batch.t_free[i], fe_min=batch.fe_min[i],
                                                        fe_max=batch.fe_max[i], rho=batch.rho[i])


def grid(edge):
    out = []
    j = 0
    while edge["fe_max"] - j * edge["rho"] >= edge["fe_min"]:
        out.append(edge["fe_max"] - j * edge["rho"])
        j += 1
    return out


def min_freq(lat_at, f_min, f_max, iters=200):
    """Smallest f in [f_min, f_max] with lat_at(f) <= 0 (lat_at decreasing in f), or None."""
    if lat_at(f_max) > 0:
        return None
    if lat_at(f_min) <= 0:
        return f_min
    lo, hi = f_min, f_max
    for _ in range(iters):
        mid = 0.5 * (lo + hi)
        if lat_at(mid) <= 0:
            hi = mid
        else:
            lo = mid
        if hi - lo <= 1e-15 * hi:
            break
    return hi


def local_energy(model, u):
    work = sum(model.g[n] * model.A[n] for n in range(1, model.N + 1))
    f = min_freq(lambda f: u["zeta"] * work / f - u["T"], u["f_min"], u["f_max"])
    assert f is not None
    return sum(u["kappa"] * model.q[n] * model.A[n] * f * f for n in range(1, model.N + 1)), f


def simulate_finish(model, users, nvec, fe, t_free, freqs):
    """As-soon-as-possible edge schedule of same-sub-task batches; returns the end of batch N."""
    N = model.N
    off = [m for m, n in enumerate(nvec) if n < N]
    nmin = min(nvec[m] for m in off)
    t = t_free
    for n in range(nmin + 1, N + 1):
        b = sum(1 for m in off if nvec[m] < n)
        ready = [t]
        for m in off:
            if nvec[m] == n - 1:
                u = users[m]
                comp = sum(u["zeta"] * model.g[k] * model.A[k] / freqs[m] for k in range(1, nvec[m] + 1))
                ready.append(comp + model.O[nvec[m]] / u["R"])
        t = max(ready) + _d(model, n, b) * model.A[n] / fe
    return t


def general_energy(model, users, edge, nvec, fe, t_free):
    """Min energy of one general candidate via bisection + ASAP simulation; None if infeasible."""
    N = model.N
    off = [m for m, n in enumerate(nvec) if n < N]
    E = 0.0
    for m, n in enumerate(nvec):
        if n == N:
            E += local_energy(model, users[m])[0]
    if not off:
        return E
    l_o = min(users[m]["T"] for m in off)
    fast = [users[m]["f_max"] for m in range(len(users))]
    if simulate_finish(model, users, nvec, fe, t_free, fast) > l_o:
        return None
    freqs = list(fast)
    for m in off:
        u = users[m]
        if nvec[m] == 0:
            freqs[m] = u["f_min"]
            continue

        def over(f, m=m):
            fr = list(fast)
            fr[m] = f
            return simulate_finish(model, users, nvec, fe, t_free, fr) - l_o

        f = min_freq(over, u["f_min"], u["f_max"])
        if f is None:
            return None
        freqs[m] = f
    # decoupling: all users at their individual minima must stay feasible
    if simulate_finish(model, users, nvec, fe, t_free, freqs) > l_o * (1 + 1e-12):
        return None
    for m in off:
        u = users[m]
        n = nvec[m]
        E += sum(u["kappa"] * model.q[k] * model.A[k] * freqs[m] ** 2 for k in range(1, n + 1))
        E += model.O[n] / u["R"] * u["p_u"]
    for n in range(1, N + 1):
        b = sum(1 for m in off if nvec[m] < n)
        if b:
            E += _c(model, n, b) * model.A[n] * fe * fe
    return E


def brute_force(batch, i, space):
    """space 0: all vectors in {0..N}^M; space 1: identical vectors {n~, N}^M (P1)."""
    model, users, edge = _inst(batch, i)
    M, N = len(users), model.N
    best = float("inf")
    fes = grid(edge)
    if space == 0:
        vecs = itertools.product(range(N + 1), repeat=M)
    else:
        vecs = set()
        for nt in range(N + 1):
            for mask in range(1 << M):
                vecs.add(tuple(nt if (nt < N and (mask >> m) & 1) else N for m in range(M)))
    for vec in vecs:
        for fe in fes:
            E = general_energy(model, users, edge, list(vec), fe, edge["t_free"])
            if E is not None and E < best:
                best = E
    return best
