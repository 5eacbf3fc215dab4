"""Seeded synthetic workload generator for the J-DOB hot path.

This module is shared INPUT plumbing: it is the only code that both the CPU
oracle (``oracle/``) and the CUDA path (``paper_2504_14611_b200``) consume.
It holds none of the method's arithmetic (no aggregates, thresholds, DVFS
closed forms, energies or argmins).  It only draws random numbers and builds
input arrays shaped like the paper's workloads; DESIGN.md §"Input recipe"
states the recipe.

Counter-based generator (DESIGN.md §Input recipe):
  mix64(x)  = SplitMix64 finaliser (add golden gamma, xor-shift-multiply x2)
  draw(seed, inst, user, field) = mix64(mix64(mix64(seed) ^ inst) ^ ((user << 8) | field))
  u01       = (draw >> 11) * 2^-53
  uniform   = lo + (hi - lo) * u01
  choice    = a + (((draw >> 32) * (b - a + 1)) >> 32)
Every draw is keyed by (seed, instance id, user, field), so any instance range
can be regenerated independently (sharding, sampled parity checks).

Paper parameters used (Table I): SNR 30 dB, W 10 MHz,
g = q = 1, p_u = 1 W, rho = 0.03 GHz, f_m in [1.5, 2.6] GHz, f_e in [0.2, 2.1] GHz,
alpha = 1, eta = 0.6.  R = W log2(1 + SNR).  beta -> T per
PAPER.md:361 ("beta = T / sum_n l^cp(f_max) - 1").
"""
from __future__ import annotations

import math
from dataclasses import dataclass, field
from typing import List, Optional, Sequence

import numpy as np

from . import profiles

U64 = np.uint64
_GOLDEN = U64(0x9E3779B97F4A7C15)
_M1 = U64(0xBF58476D1CE4E5B9)
_M2 = U64(0x94D049BB133111EB)

# field ids of the counter-based draws
F_M, F_MODEL, F_REGIME, F_RHO, F_BETA_USER, F_BETA_INST, F_R_HET, F_K_HET, F_TFREE = range(9)


def mix64(x):
    """SplitMix64 finaliser on a uint64 numpy array (wrapping arithmetic)."""
    x = np.asarray(x, dtype=U64)
    with np.errstate(over="ignore"):
        x = x + _GOLDEN
        x = (x ^ (x >> U64(30))) * _M1
        x = (x ^ (x >> U64(27))) * _M2
    return x ^ (x >> U64(31))


def draw(seed, inst, user, fld):
    seed = np.asarray(seed, dtype=U64)
    inst = np.asarray(inst, dtype=U64)
    user = np.asarray(user, dtype=U64)
    fld = np.asarray(fld, dtype=U64)
    return mix64(mix64(mix64(seed) ^ inst) ^ ((user << U64(8)) | fld))


def u01(d):
    return (np.asarray(d, dtype=U64) >> U64(11)).astype(np.float64) * (2.0 ** -53)


def uniform(d, lo, hi):
    return lo + (hi - lo) * u01(d)


def choice(d, a, b):
    """Integer in [a, b] from the top 32 bits (Lemire-style multiply-shift)."""
    hi = (np.asarray(d, dtype=U64) >> U64(32))
    with np.errstate(over="ignore"):
        return a + ((hi * U64(b - a + 1)) >> U64(32)).astype(np.int64)


# --------------------------------------------------------------------------------------
# Containers
# --------------------------------------------------------------------------------------
@dataclass
class Model:
    """One DNN profile (§II-B lines 92-94, Eq. (5)).

    A, O, g, q have N+1 entries (index 0 is the virtual input layer, A[0] = 0).
    d, c are row-major [(N+1) x (B_max+1)] tables, element n*(B_max+1)+b.
    """
    name: str
    N: int
    B_max: int
    A: np.ndarray
    O: np.ndarray
    g: np.ndarray
    q: np.ndarray
    d: np.ndarray
    c: np.ndarray

    def table(self, t, n, b):
        return float(t[n * (self.B_max + 1) + b])


@dataclass
class Batch:
    """CSR batch of independent instances (DESIGN.md §Data layout)."""
    models: List[Model]
    model_id: np.ndarray            # int32 [n_inst]
    user_off: np.ndarray            # int64 [n_inst+1]
    zeta: np.ndarray                # float64 [n_users] ...
    kappa: np.ndarray
    f_min: np.ndarray
    f_max: np.ndarray
    R: np.ndarray
    p_u: np.ndarray
    T: np.ndarray
    t_free: np.ndarray              # float64 [n_inst]
    fe_min: np.ndarray
    fe_max: np.ndarray
    rho: np.ndarray
    bucket: Optional[np.ndarray] = None   # int32 [n_inst] statistics bucket (a12), optional
    inst_base: int = 0              # global id of instance 0 (for regeneration)
    meta: dict = field(default_factory=dict)

    USER_FIELDS = ("zeta", "kappa", "f_min", "f_max", "R", "p_u", "T")
    INST_FIELDS = ("t_free", "fe_min", "fe_max", "rho")

    @property
    def n_inst(self) -> int:
        return int(self.model_id.shape[0])

    @property
    def n_users(self) -> int:
        return int(self.user_off[-1])

    def M(self, i: int) -> int:
        return int(self.user_off[i + 1] - self.user_off[i])

    def subset(self, i0: int, i1: int) -> "Batch":
        o0, o1 = int(self.user_off[i0]), int(self.user_off[i1])
        kw = {f: getattr(self, f)[o0:o1].copy() for f in self.USER_FIELDS}
        kw.update({f: getattr(self, f)[i0:i1].copy() for f in self.INST_FIELDS})
        return Batch(models=self.models, model_id=self.model_id[i0:i1].copy(),
                     user_off=(self.user_off[i0:i1 + 1] - o0).astype(np.int64),
                     bucket=None if self.bucket is None else self.bucket[i0:i1].copy(),
                     inst_base=self.inst_base + i0, meta=dict(self.meta), **kw)

    def take(self, idx: Sequence[int]) -> "Batch":
        """Gather an arbitrary list of instances into a new batch."""
        idx = np.asarray(idx, dtype=np.int64)
        parts = [np.arange(self.user_off[i], self.user_off[i + 1]) for i in idx]
        uidx = np.concatenate(parts) if parts else np.zeros(0, np.int64)
        Ms = np.array([self.M(int(i)) for i in idx], dtype=np.int64)
        off = np.zeros(len(idx) + 1, np.int64)
        off[1:] = np.cumsum(Ms)
        kw = {f: getattr(self, f)[uidx].copy() for f in self.USER_FIELDS}
        kw.update({f: getattr(self, f)[idx].copy() for f in self.INST_FIELDS})
        return Batch(models=self.models, model_id=self.model_id[idx].copy(), user_off=off,
                     bucket=None if self.bucket is None else self.bucket[idx].copy(),
                     inst_base=0, meta=dict(self.meta, taken=True), **kw)

    def nbytes(self) -> int:
        n = self.model_id.nbytes + self.user_off.nbytes
        n += sum(getattr(self, f).nbytes for f in self.USER_FIELDS + self.INST_FIELDS)
        if self.bucket is not None:
            n += self.bucket.nbytes
        return n


def concat(batches: Sequence[Batch]) -> Batch:
    """Concatenate batches; model lists are shared when identical, else appended (model_id shifted)."""
    models = batches[0].models
    shared = all(b.models is models for b in batches)
    if not shared:
        models = [m for b in batches for m in b.models]
    offs = [np.zeros(1, np.int64)]
    mids = []
    base = 0
    mbase = 0
    for b in batches:
        offs.append(b.user_off[1:] + base)
        base += b.n_users
        mids.append(b.model_id + (0 if shared else mbase))
        mbase += len(b.models)
    kw = {f: np.concatenate([getattr(b, f) for b in batches]) for f in Batch.USER_FIELDS + Batch.INST_FIELDS}
    bucket = None
    if all(b.bucket is not None for b in batches):
        bucket = np.concatenate([b.bucket for b in batches])
    return Batch(models=models, model_id=np.concatenate(mids).astype(np.int32),
                 user_off=np.concatenate(offs), bucket=bucket, **kw)


# --------------------------------------------------------------------------------------
# Table I defaults
# --------------------------------------------------------------------------------------
TABLE_I = dict(snr_db=30.0, W=10e6, p_u=1.0, rho=0.03e9, f_min=1.5e9, f_max=2.6e9,
               fe_min=0.2e9, fe_max=2.1e9, alpha=1.0, eta=0.6)


def rate(W: float, snr_db: float) -> float:
    """R = W log2(1 + SNR). Host-side input preparation only."""
    return W * math.log2(1.0 + 10.0 ** (snr_db / 10.0))


R_TABLE_I = rate(TABLE_I["W"], TABLE_I["snr_db"])


def min_local_latency(model: Model, zeta: np.ndarray, f_max: np.ndarray) -> np.ndarray:
    """zeta * sum_n g_n A_n / f_max, the beta denominator of PAPER.md:361.

    Input recipe only (deadline synthesis); summation ascending in n."""
    s = 0.0
    for n in range(0, model.N + 1):
        s = s + float(model.g[n]) * float(model.A[n])
    return (zeta * s) / f_max


def deadline_from_beta(model: Model, zeta, f_max, beta):
    """T = (1 + beta) * (zeta v_N / f_max)  (PAPER.md:361 inverted)."""
    return (1.0 + np.asarray(beta, np.float64)) * min_local_latency(model, np.asarray(zeta, np.float64),
                                                                    np.asarray(f_max, np.float64))


# --------------------------------------------------------------------------------------
# Builders
# --------------------------------------------------------------------------------------
def _batch_from_lists(models, model_id, Ms, user_cols, inst_cols, bucket=None, inst_base=0, meta=None):
    off = np.zeros(len(Ms) + 1, np.int64)
    off[1:] = np.cumsum(np.asarray(Ms, np.int64))
    kw = {f: np.ascontiguousarray(np.asarray(user_cols[f], np.float64)) for f in Batch.USER_FIELDS}
    kw.update({f: np.ascontiguousarray(np.asarray(inst_cols[f], np.float64)) for f in Batch.INST_FIELDS})
    return Batch(models=list(models), model_id=np.asarray(model_id, np.int32), user_off=off,
                 bucket=None if bucket is None else np.asarray(bucket, np.int32),
                 inst_base=inst_base, meta=meta or {}, **kw)


def single_instance(model: Model, users: dict, t_free=0.0, fe_min=0.2e9, fe_max=2.1e9, rho=0.03e9) -> Batch:
    M = len(users["T"])
    cols = {f: np.broadcast_to(np.asarray(users[f], np.float64), (M,)).copy() for f in Batch.USER_FIELDS}
    inst = dict(t_free=[t_free], fe_min=[fe_min], fe_max=[fe_max], rho=[rho])
    return _batch_from_lists([model], [0], [M], cols, inst)


def toy_instance(name: str) -> Batch:
    """SPEC.md:204 toys ("toy-1", "toy-2") and SURVEY Appendix C variants / C1 (toy-4)."""
    base_users = dict(zeta=1.0, kappa=1e-27, f_min=1.5e9, f_max=2.6e9, R=1e8, p_u=1.0)
    if name in ("toy-1", "toy-2", "toy-2-m1", "toy-2-tfree"):
        m = profiles.toy1() if name == "toy-1" else profiles.toy2()
        T = [0.2] if name == "toy-2-m1" else [0.2, 0.25]
        users = dict(base_users, T=T)
        t_free = 0.196 if name == "toy-2-tfree" else 0.0
        return single_instance(m, users, t_free=t_free)
    if name == "toy-4":
        users = dict(base_users, T=[0.3, 0.3])
        return single_instance(profiles.toy4(), users, t_free=0.0, fe_min=0.2e9, fe_max=2.1e9, rho=0.95e9)
    raise KeyError(name)


def _table_i_users(n_users, zeta, kappa):
    return dict(zeta=np.full(n_users, zeta), kappa=np.full(n_users, kappa),
                f_min=np.full(n_users, TABLE_I["f_min"]), f_max=np.full(n_users, TABLE_I["f_max"]),
                R=np.full(n_users, R_TABLE_I), p_u=np.full(n_users, TABLE_I["p_u"]))


def config_c2(n_inst: int = 1 << 20, seed: int = 2, inst_begin: int = 0) -> Batch:
    """C2: 10 homogeneous Table-I users, VGG-16-like profile, identical deadlines,
    per-instance beta ~ U[0, 35] (covers the paper's 2.13 and 30.25)."""
    model = profiles.vgg16()
    M = 10
    ids = np.arange(inst_begin, inst_begin + n_inst, dtype=np.int64)
    beta = uniform(draw(seed, ids, 0, F_BETA_INST), 0.0, 35.0)
    zeta, kappa = profiles.ZETA, profiles.KAPPA
    T_inst = deadline_from_beta(model, zeta, TABLE_I["f_max"], beta)
    users = _table_i_users(n_inst * M, zeta, kappa)
    users["T"] = np.repeat(T_inst, M)
    inst = dict(t_free=np.zeros(n_inst), fe_min=np.full(n_inst, TABLE_I["fe_min"]),
                fe_max=np.full(n_inst, TABLE_I["fe_max"]), rho=np.full(n_inst, TABLE_I["rho"]))
    bucket = np.minimum((beta / 5.0).astype(np.int32), 6)          # 7 beta bands of width 5
    return _batch_from_lists([model], np.zeros(n_inst, np.int32), np.full(n_inst, M), users, inst,
                             bucket=bucket, inst_base=inst_begin,
                             meta=dict(config="c2", seed=seed, n_buckets=7))


C3_BETA_RANGES = ((4.5, 5.5), (2.0, 8.0), (0.0, 10.0))


def config_c3(n_inst: int = 100_000, seed: int = 3, inst_begin: int = 0) -> Batch:
    """C3: ResNet-18-like, M ~ U{4..20}, per-user beta ~ U[lo, hi] cycling through the
    paper's three ranges, deadlines i.i.d.."""
    model = profiles.resnet18()
    ids = np.arange(inst_begin, inst_begin + n_inst, dtype=np.int64)
    Ms = choice(draw(seed, ids, 0, F_M), 4, 20)
    off = np.zeros(n_inst + 1, np.int64)
    off[1:] = np.cumsum(Ms)
    n_users = int(off[-1])
    inst_of_user = np.repeat(ids, Ms)
    user_idx = np.arange(n_users, dtype=np.int64) - np.repeat(off[:-1], Ms)
    rng = np.array(C3_BETA_RANGES)
    regime = (ids % 3).astype(np.int64)
    lo = np.repeat(rng[regime, 0], Ms)
    hi = np.repeat(rng[regime, 1], Ms)
    beta = uniform(draw(seed, inst_of_user, user_idx, F_BETA_USER), lo, hi)
    zeta, kappa = profiles.ZETA, profiles.KAPPA
    users = _table_i_users(n_users, zeta, kappa)
    users["T"] = deadline_from_beta(model, zeta, TABLE_I["f_max"], beta)
    inst = dict(t_free=np.zeros(n_inst), fe_min=np.full(n_inst, TABLE_I["fe_min"]),
                fe_max=np.full(n_inst, TABLE_I["fe_max"]), rho=np.full(n_inst, TABLE_I["rho"]))
    return _batch_from_lists([model], np.zeros(n_inst, np.int32), Ms, users, inst,
                             bucket=regime.astype(np.int32), inst_base=inst_begin,
                             meta=dict(config="c3", seed=seed, n_buckets=3))


def config_c4(seed: int = 4) -> Batch:
    """C4: one ResNet-18-like instance, M = 8, beta_m ~ U[2, 8], Table I grid (k = 64)."""
    model = profiles.resnet18()
    M = 8
    beta = uniform(draw(seed, 0, np.arange(M), F_BETA_USER), 2.0, 8.0)
    zeta, kappa = profiles.ZETA, profiles.KAPPA
    users = _table_i_users(M, zeta, kappa)
    users["T"] = deadline_from_beta(model, zeta, TABLE_I["f_max"], beta)
    inst = dict(t_free=[0.0], fe_min=[TABLE_I["fe_min"]], fe_max=[TABLE_I["fe_max"]], rho=[TABLE_I["rho"]])
    return _batch_from_lists([model], [0], [M], users, inst, meta=dict(config="c4", seed=seed))


C5_REGIMES = ("ident_2.13", "ident_30.25", "mixed_4.5_5.5", "mixed_2_8", "mixed_0_10")
C5_RHOS = (1e7, 3e7, 1e8)


def config_c5(n_inst: int = 10_000_000, seed: int = 5, inst_begin: int = 0, hetero: bool = False) -> Batch:
    """C5 Monte Carlo: M ~ U{1..32}; model in {MobileNetV2, VGG-16, ResNet-18};
    regime in {identical beta 2.13, identical 30.25, mixed U[4.5,5.5], U[2,8], U[0,10]};
    rho in {10, 30, 100} MHz.  Optional heterogeneity R x U[0.5,2], kappa x U[0.5,2]."""
    models = [profiles.mobilenetv2(), profiles.vgg16(), profiles.resnet18()]
    ids = np.arange(inst_begin, inst_begin + n_inst, dtype=np.int64)
    Ms = choice(draw(seed, ids, 0, F_M), 1, 32)
    mid = choice(draw(seed, ids, 0, F_MODEL), 0, 2)
    regime = choice(draw(seed, ids, 0, F_REGIME), 0, 4)
    rho = np.array(C5_RHOS)[choice(draw(seed, ids, 0, F_RHO), 0, 2)]
    off = np.zeros(n_inst + 1, np.int64)
    off[1:] = np.cumsum(Ms)
    n_users = int(off[-1])
    inst_of_user = np.repeat(ids, Ms)
    local = np.repeat(np.arange(n_inst, dtype=np.int64), Ms)
    user_idx = np.arange(n_users, dtype=np.int64) - np.repeat(off[:-1], Ms)
    reg_u = regime[local]
    lo = np.choose(reg_u, [2.13, 30.25, 4.5, 2.0, 0.0])
    hi = np.choose(reg_u, [2.13, 30.25, 5.5, 8.0, 10.0])
    beta_user = uniform(draw(seed, inst_of_user, user_idx, F_BETA_USER), lo, hi)
    beta = np.where(reg_u < 2, lo, beta_user)
    zeta, kappa = profiles.ZETA, profiles.KAPPA
    users = _table_i_users(n_users, zeta, kappa)
    if hetero:
        users["R"] = users["R"] * uniform(draw(seed, inst_of_user, user_idx, F_R_HET), 0.5, 2.0)
        users["kappa"] = users["kappa"] * uniform(draw(seed, inst_of_user, user_idx, F_K_HET), 0.5, 2.0)
    lat = np.empty(n_users)
    mid_u = mid[local]
    for k, m in enumerate(models):
        sel = mid_u == k
        lat[sel] = min_local_latency(m, users["zeta"][sel], users["f_max"][sel])
    users["T"] = (1.0 + beta) * lat
    inst = dict(t_free=np.zeros(n_inst), fe_min=np.full(n_inst, TABLE_I["fe_min"]),
                fe_max=np.full(n_inst, TABLE_I["fe_max"]), rho=rho)
    # statistics buckets by (model, deadline regime, M) -- SURVEY §8(a) a12: 3 x 5 x 32 = 480
    bucket = ((mid * 5 + regime) * 32 + (Ms - 1)).astype(np.int32)
    return _batch_from_lists(models, mid.astype(np.int32), Ms, users, inst, bucket=bucket,
                             inst_base=inst_begin, meta=dict(config="c5", seed=seed, n_buckets=480))


def c5_device_inputs(seed: int = 5, inst_begin: int = 0, hetero: bool = False):
    """(models, params) for the device twin of config_c5 (include/jdob.h jdob_gen_params): the recipe's
    constants as the doubles config_c5 uses -- Table I users and, per model, the beta denominator
    zeta v_N / f_max of the homogeneous users (min_local_latency on one user)."""
    models = [profiles.mobilenetv2(), profiles.vgg16(), profiles.resnet18()]
    zeta, kappa = profiles.ZETA, profiles.KAPPA
    lat = [float(min_local_latency(m, np.array([zeta]), np.array([TABLE_I["f_max"]]))[0]) for m in models]
    params = dict(seed=seed, inst_begin=inst_begin, hetero=int(hetero), zeta=zeta, kappa=kappa,
                  f_min=TABLE_I["f_min"], f_max=TABLE_I["f_max"], R=R_TABLE_I, p_u=TABLE_I["p_u"],
                  fe_min=TABLE_I["fe_min"], fe_max=TABLE_I["fe_max"], rho=list(C5_RHOS), lat=lat)
    return models, params


def random_batch(seed: int, n_inst: int, M_lo: int = 1, M_hi: int = 8, N_lo: int = 1, N_hi: int = 6,
                 tfree_frac: float = 0.3, k_max: int = 40, B_extra: int = 2, identical_T_frac: float = 0.3,
                 equal_gamma_frac: float = 0.3) -> Batch:
    """Heterogeneous random stress instances, each with its own random model.

    Used by the property and parity tests (small M, N).  Deadlines are drawn as
    beta in [0, 10] over the minimum local latency, so every user is locally
    feasible; a fraction of instances gets t_free > 0 but never
    above min T (the Require of Alg. 1)."""
    models = []
    cols = {f: [] for f in Batch.USER_FIELDS}
    inst = {f: [] for f in Batch.INST_FIELDS}
    Ms = []
    for i in range(n_inst):
        def dr(user, fld):
            return draw(seed, i, user, fld)
        def un(user, fld, lo, hi):
            return float(uniform(dr(user, fld), lo, hi))
        def ch(user, fld, a, b):
            return int(choice(dr(user, fld), a, b))
        M = ch(0, 0, M_lo, M_hi)
        N = ch(0, 1, N_lo, N_hi)
        B_max = min(32, M + ch(0, 2, 0, B_extra))
        A = [0.0] + [float(round(un(n, 10, 0.2, 3.0) * 1e8)) for n in range(1, N + 1)]
        O = [float(round(un(n, 11, 0.05, 1.5) * 1e6)) for n in range(0, N + 1)]
        g = [1.0] * (N + 1)
        q = [1.0] * (N + 1)
        d = np.zeros((N + 1) * (B_max + 1))
        c = np.zeros((N + 1) * (B_max + 1))
        for n in range(1, N + 1):
            d1 = un(n, 12, 0.3, 1.2)
            c1 = un(n, 13, 0.5, 5.0) * 1e-29 * (10.0 ** ch(n, 16, -1, 2))
            sig_d = un(n, 14, 0.05, 1.0)
            sig_c = un(n, 15, 0.05, 1.0)
            for b in range(1, B_max + 1):
                d[n * (B_max + 1) + b] = d1 * (1.0 + sig_d * (b - 1))
                c[n * (B_max + 1) + b] = c1 * (1.0 + sig_c * (b - 1))
        model = Model(f"rand{i}", N, B_max, np.array(A), np.array(O), np.array(g), np.array(q), d, c)
        models.append(model)
        same_gamma = un(0, 3, 0.0, 1.0) < equal_gamma_frac
        same_T = un(0, 4, 0.0, 1.0) < identical_T_frac
        for m in range(M):
            mm = 0 if same_gamma else m
            zeta = un(mm, 20, 0.5, 1.5)
            kappa = un(m, 21, 0.5, 2.0) * 1e-27
            f_min = float(round(un(mm, 22, 1.0, 1.6), 2) * 1e9)
            f_max = float(round(un(mm, 23, 2.0, 3.0), 2) * 1e9)
            R = float(round(un(mm, 24, 0.5, 2.0) * 1e8))
            p_u = un(m, 25, 0.5, 1.5)
            beta = un(0 if same_T else m, 26, 0.0, 10.0)
            lat = float(min_local_latency(model, np.array([zeta]), np.array([f_max]))[0])
            T = (1.0 + beta) * lat
            for f, v in zip(Batch.USER_FIELDS, (zeta, kappa, f_min, f_max, R, p_u, T)):
                cols[f].append(v)
        Ts = cols["T"][-M:]
        t_free = 0.0
        if un(0, 5, 0.0, 1.0) < tfree_frac:
            t_free = un(0, 6, 0.0, 0.9) * min(Ts)
        fe_max = float(round(un(0, 7, 1.5, 2.5), 2) * 1e9)
        fe_min = float(round(un(0, 8, 0.1, 0.5), 2) * 1e9)
        k = ch(0, 9, 1, k_max)
        rho = float(round((fe_max - fe_min) / max(k - 1, 1) / 1e6) * 1e6) if k > 1 else fe_max
        for f, v in zip(Batch.INST_FIELDS, (t_free, fe_min, fe_max, rho)):
            inst[f].append(v)
        Ms.append(M)
    return _batch_from_lists(models, np.arange(n_inst), Ms, cols, inst, meta=dict(config="random", seed=seed))


def grid_size(fe_min: float, fe_max: float, rho: float) -> int:
    """Number of points f_e(j) = fe_max - j*rho with f_e(j) >= fe_min (DESIGN reading R7).

    Input-side helper for sizing index spaces (the same rule both solvers apply)."""
    k = 0
    while fe_max - float(k) * rho >= fe_min:
        k += 1
    return k


def config_batch(name: str, n_inst: Optional[int] = None, seed: Optional[int] = None, inst_begin: int = 0) -> Batch:
    name = name.lower()
    if name in ("c1", "toy-4"):
        return toy_instance("toy-4")
    if name == "c2":
        return config_c2(n_inst if n_inst is not None else 1 << 20, 2 if seed is None else seed, inst_begin)
    if name == "c3":
        return config_c3(n_inst if n_inst is not None else 100_000, 3 if seed is None else seed, inst_begin)
    if name == "c4":
        return config_c4(4 if seed is None else seed)
    if name == "c5":
        return config_c5(n_inst if n_inst is not None else 10_000_000, 5 if seed is None else seed, inst_begin)
    raise KeyError(name)
