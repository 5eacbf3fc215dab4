"""ctypes wrapper around the plain C oracle (oracle/jdob_oracle.c).

TEST INFRASTRUCTURE ONLY: importable by tests/, __graft_entry__.smoke() and the
cpu_baseline / --impl reference legs of bench.py.  The product package
(paper_2504_14611_b200) never imports this module.
"""
from __future__ import annotations

import ctypes as C
import os
import subprocess
import threading

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
SRC = os.path.join(HERE, "jdob_oracle.c")
LIB = os.path.join(HERE, "liboracle.so")
# tools/mutate_oracle.py points this at a mutated build (mutation testing of the pins)
LIB_OVERRIDE = os.environ.get("JDOB_ORACLE_LIB")
CFLAGS = ["-O2", "-std=gnu11", "-ffp-contract=off", "-fno-fast-math", "-fPIC", "-shared", "-pthread", "-Wall"]

ST_OK, ST_LOCAL_INFEASIBLE, ST_REQUIRE, ST_BADPARAM, ST_BADMODEL, ST_TOOBIG = range(6)
STATS_FIELDS = 80
MODE_FULL, MODE_LC, MODE_NO_EDGE_DVFS, MODE_BINARY = range(4)
MAXM_LARGE = 1024

_lock = threading.Lock()
_lib = None


def build(force: bool = False) -> str:
    """Compile the oracle with gcc (IEEE binary64, no FMA contraction)."""
    if force or not os.path.exists(LIB) or os.path.getmtime(LIB) < os.path.getmtime(SRC):
        tmp = LIB + f".tmp{os.getpid()}"
        subprocess.check_call(["gcc", *CFLAGS, "-o", tmp, SRC, "-lm"])
        os.replace(tmp, LIB)
    return LIB


class OModel(C.Structure):
    _fields_ = [("N", C.c_int), ("B_max", C.c_int),
                ("A", C.POINTER(C.c_double)), ("O", C.POINTER(C.c_double)),
                ("g", C.POINTER(C.c_double)), ("q", C.POINTER(C.c_double)),
                ("d", C.POINTER(C.c_double)), ("c", C.POINTER(C.c_double))]


class OInst(C.Structure):
    _fields_ = [("M", C.c_int)] + [(f, C.POINTER(C.c_double)) for f in
                                   ("zeta", "kappa", "f_min", "f_max", "R", "p_u", "T")] + \
               [(f, C.c_double) for f in ("t_free", "fe_min", "fe_max", "rho")]


class OResult(C.Structure):
    _fields_ = [("E", C.c_double), ("E_lc", C.c_double), ("t_free_next", C.c_double), ("f_e", C.c_double),
                ("n_tilde", C.c_int), ("j", C.c_int), ("status", C.c_int), ("mask", C.c_uint),
                ("f_user", C.c_double * MAXM_LARGE), ("part", C.c_int * MAXM_LARGE),
                ("n_visit", C.c_longlong), ("n_eval", C.c_longlong), ("n_member", C.c_longlong)]


class OOgResult(C.Structure):
    _fields_ = [("E", C.c_double), ("t_free_next", C.c_double), ("status", C.c_int), ("n_groups", C.c_int),
                ("group_of", C.c_int * MAXM_LARGE), ("part", C.c_int * MAXM_LARGE),
                ("f_user", C.c_double * MAXM_LARGE),
                ("group_fe", C.c_double * 32), ("group_start", C.c_int * 33)]


class OBatch(C.Structure):
    _fields_ = [("models", C.POINTER(OModel)), ("model_id", C.POINTER(C.c_int)),
                ("user_off", C.POINTER(C.c_longlong))] + \
               [(f, C.POINTER(C.c_double)) for f in
                ("zeta", "kappa", "f_min", "f_max", "R", "p_u", "T", "t_free", "fe_min", "fe_max", "rho")]


class OOut(C.Structure):
    _fields_ = [(f, C.POINTER(C.c_double)) for f in ("E", "E_lc", "t_free_next", "f_e", "f_user")] + \
               [(f, C.POINTER(C.c_int)) for f in ("n_tilde", "j", "status")] + \
               [("mask", C.POINTER(C.c_uint)), ("counts", C.POINTER(C.c_longlong)), ("part", C.POINTER(C.c_int))]


def lib():
    global _lib
    with _lock:
        if _lib is None:
            if LIB_OVERRIDE:
                L = C.CDLL(LIB_OVERRIDE)
            else:
                build()
                L = C.CDLL(LIB)
            P = C.POINTER
            L.oracle_check_model.argtypes = [P(OModel)]
            L.oracle_check_inst.argtypes = [P(OModel), P(OInst)]
            L.oracle_lc.argtypes = [P(OModel), P(OInst), P(C.c_double), P(C.c_double)]
            L.oracle_lc.restype = C.c_double
            L.oracle_thresholds.argtypes = [P(OModel), P(OInst), C.c_int, P(C.c_double), P(C.c_int), P(C.c_double)]
            L.oracle_thresholds.restype = None
            L.oracle_jdob.argtypes = [P(OModel), P(OInst), C.c_int, P(OResult)]
            L.oracle_bf.argtypes = [P(OModel), P(OInst), C.c_int, C.c_ulonglong, C.c_ulonglong,
                                    P(C.c_double), P(C.c_longlong)]
            L.oracle_bf_mt.argtypes = [P(OModel), P(OInst), C.c_int, C.c_ulonglong, C.c_ulonglong, C.c_int,
                                       P(C.c_double), P(C.c_longlong)]
            L.oracle_bf_candidate.argtypes = [P(OModel), P(OInst), C.c_int, C.c_ulonglong]
            L.oracle_bf_candidate.restype = C.c_double
            L.oracle_bf_space_size.argtypes = [P(OModel), P(OInst), C.c_int]
            L.oracle_bf_space_size.restype = C.c_ulonglong
            L.oracle_eval.argtypes = [P(OModel), P(OInst), P(C.c_int), C.c_double, C.c_double, P(C.c_double),
                                      P(C.c_double), P(C.c_double), P(C.c_uint)]
            L.oracle_solve_batch.argtypes = [P(OBatch), C.c_longlong, C.c_int, P(OOut), C.c_int]
            L.oracle_eval_batch.argtypes = [P(OBatch), C.c_longlong, P(C.c_int), P(C.c_double), C.c_double,
                                            P(C.c_double), P(C.c_double), P(C.c_double), P(C.c_uint),
                                            P(C.c_int)]
            L.oracle_stats.argtypes = [C.c_longlong, P(C.c_longlong), P(C.c_int), C.c_int, P(C.c_double),
                                       P(C.c_double), P(C.c_int), P(C.c_double), P(C.c_int), P(C.c_double)]
            L.oracle_grid_k.argtypes = [P(OInst)]
            L.oracle_og.argtypes = [P(OModel), P(OInst), C.c_int, P(OOgResult)]
            _lib = L
    return _lib


def _dp(a):
    return a.ctypes.data_as(C.POINTER(C.c_double))


def _ip(a):
    return a.ctypes.data_as(C.POINTER(C.c_int))


class _Keep:
    """Holds numpy arrays alive while ctypes structs point into them."""

    def __init__(self):
        self.refs = []

    def f64(self, x):
        a = np.ascontiguousarray(np.asarray(x, dtype=np.float64))
        self.refs.append(a)
        return a


def _omodel(model, keep):
    s = OModel()
    s.N, s.B_max = int(model.N), int(model.B_max)
    for f in ("A", "O", "g", "q", "d", "c"):
        setattr(s, f, _dp(keep.f64(getattr(model, f))))
    return s


def _oinst(batch, i, keep):
    o0, o1 = int(batch.user_off[i]), int(batch.user_off[i + 1])
    s = OInst()
    s.M = o1 - o0
    for f in ("zeta", "kappa", "f_min", "f_max", "R", "p_u", "T"):
        setattr(s, f, _dp(keep.f64(getattr(batch, f)[o0:o1])))
    for f in ("t_free", "fe_min", "fe_max", "rho"):
        setattr(s, f, float(getattr(batch, f)[i]))
    return s


def _obatch(batch, keep):
    models = (OModel * len(batch.models))(*[_omodel(m, keep) for m in batch.models])
    keep.refs.append(models)
    s = OBatch()
    s.models = C.cast(models, C.POINTER(OModel))
    mid = np.ascontiguousarray(batch.model_id, dtype=np.int32)
    off = np.ascontiguousarray(batch.user_off, dtype=np.int64)
    keep.refs += [mid, off]
    s.model_id = _ip(mid)
    s.user_off = off.ctypes.data_as(C.POINTER(C.c_longlong))
    for f in ("zeta", "kappa", "f_min", "f_max", "R", "p_u", "T", "t_free", "fe_min", "fe_max", "rho"):
        setattr(s, f, _dp(keep.f64(getattr(batch, f))))
    return s


# ------------------------------------------------------------------------------------
# Public helpers
# ------------------------------------------------------------------------------------
def check_model(model) -> int:
    keep = _Keep()
    return lib().oracle_check_model(C.byref(_omodel(model, keep)))


def check_inst(batch, i=0) -> int:
    keep = _Keep()
    return lib().oracle_check_inst(C.byref(_omodel(batch.models[batch.model_id[i]], keep)),
                                   C.byref(_oinst(batch, i, keep)))


def lc(batch, i=0):
    keep = _Keep()
    M = batch.M(i)
    f = np.zeros(M)
    e = np.zeros(M)
    E = lib().oracle_lc(C.byref(_omodel(batch.models[batch.model_id[i]], keep)), C.byref(_oinst(batch, i, keep)),
                        _dp(f), _dp(e))
    return E, f, e


def thresholds(batch, i, nt):
    keep = _Keep()
    M = batch.M(i)
    gam = np.zeros(M)
    lst = np.zeros(M, np.int32)
    th = np.zeros(M)
    lib().oracle_thresholds(C.byref(_omodel(batch.models[batch.model_id[i]], keep)),
                            C.byref(_oinst(batch, i, keep)), nt, _dp(gam), _ip(lst), _dp(th))
    return gam, lst, th


def jdob(batch, i=0, mode=MODE_FULL) -> dict:
    keep = _Keep()
    r = OResult()
    lib().oracle_jdob(C.byref(_omodel(batch.models[batch.model_id[i]], keep)), C.byref(_oinst(batch, i, keep)),
                      mode, C.byref(r))
    M = batch.M(i)
    return dict(E=r.E, E_lc=r.E_lc, t_free_next=r.t_free_next, f_e=r.f_e, n_tilde=r.n_tilde, j=r.j,
                status=r.status, mask=r.mask, f_user=np.array(r.f_user[:M]), part=np.array(r.part[:M]),
                n_visit=r.n_visit, n_eval=r.n_eval, n_member=r.n_member)


def solve_batch(batch, mode=MODE_FULL, threads=1, counts=False) -> dict:
    keep = _Keep()
    n = batch.n_inst
    out = dict(E=np.zeros(n), E_lc=np.zeros(n), t_free_next=np.zeros(n), f_e=np.zeros(n),
               f_user=np.zeros(batch.n_users), n_tilde=np.zeros(n, np.int32), j=np.zeros(n, np.int32),
               status=np.zeros(n, np.int32), mask=np.zeros(n, np.uint32), part=np.zeros(batch.n_users, np.int32))
    if counts:
        out["counts"] = np.zeros((n, 3), np.int64)
    o = OOut()
    for f in ("E", "E_lc", "t_free_next", "f_e", "f_user"):
        setattr(o, f, _dp(out[f]))
    for f in ("n_tilde", "j", "status"):
        setattr(o, f, _ip(out[f]))
    o.mask = out["mask"].ctypes.data_as(C.POINTER(C.c_uint))
    o.counts = out["counts"].ctypes.data_as(C.POINTER(C.c_longlong)) if counts else None
    o.part = _ip(out["part"])
    b = _obatch(batch, keep)
    lib().oracle_solve_batch(C.byref(b), n, mode, C.byref(o), int(threads))
    return out


def bf_space_size(batch, space, i=0) -> int:
    keep = _Keep()
    return int(lib().oracle_bf_space_size(C.byref(_omodel(batch.models[batch.model_id[i]], keep)),
                                          C.byref(_oinst(batch, i, keep)), space))


def bf(batch, space, begin=0, end=None, threads=1, i=0):
    """Argmin (E, idx) over the candidate range [begin, end) of instance i."""
    keep = _Keep()
    if end is None:
        end = bf_space_size(batch, space, i)
    E = C.c_double()
    idx = C.c_longlong()
    m = _omodel(batch.models[batch.model_id[i]], keep)
    ins = _oinst(batch, i, keep)
    if threads <= 1:
        st = lib().oracle_bf(C.byref(m), C.byref(ins), space, begin, end, C.byref(E), C.byref(idx))
    else:
        st = lib().oracle_bf_mt(C.byref(m), C.byref(ins), space, begin, end, threads, C.byref(E), C.byref(idx))
    return E.value, idx.value, st


def bf_candidate(batch, space, idx, i=0) -> float:
    keep = _Keep()
    return lib().oracle_bf_candidate(C.byref(_omodel(batch.models[batch.model_id[i]], keep)),
                                     C.byref(_oinst(batch, i, keep)), space, int(idx))


def grid_k(batch, i=0) -> int:
    keep = _Keep()
    return lib().oracle_grid_k(C.byref(_oinst(batch, i, keep)))


def eval_config(batch, i, nvec, fe, slack=1e-9):
    keep = _Keep()
    M = batch.M(i)
    nv = np.ascontiguousarray(np.asarray(nvec, np.int32))
    E = C.c_double()
    tf = C.c_double()
    fs = np.zeros(M)
    v = C.c_uint()
    st = lib().oracle_eval(C.byref(_omodel(batch.models[batch.model_id[i]], keep)), C.byref(_oinst(batch, i, keep)),
                           _ip(nv), float(fe), float(slack), C.byref(E), C.byref(tf), _dp(fs), C.byref(v))
    return dict(E=E.value, t_free_next=tf.value, f_user=fs, violations=v.value, status=st)


def eval_batch(batch, partition, fe, slack=1e-9) -> dict:
    keep = _Keep()
    n = batch.n_inst
    part = np.ascontiguousarray(np.asarray(partition, np.int32))
    fe = np.ascontiguousarray(np.asarray(fe, np.float64))
    out = dict(E=np.zeros(n), t_free_next=np.zeros(n), f_user=np.zeros(batch.n_users),
               violations=np.zeros(n, np.uint32), status=np.zeros(n, np.int32))
    b = _obatch(batch, keep)
    lib().oracle_eval_batch(C.byref(b), n, _ip(part), _dp(fe), float(slack), _dp(out["E"]),
                            _dp(out["t_free_next"]), _dp(out["f_user"]),
                            out["violations"].ctypes.data_as(C.POINTER(C.c_uint)), _ip(out["status"]))
    return out


def stats(batch, res, n_buckets=None) -> np.ndarray:
    n = batch.n_inst
    bucket = batch.bucket
    if n_buckets is None:
        n_buckets = int(batch.meta.get("n_buckets", 32)) if bucket is not None else 32
    st = np.zeros((n_buckets, STATS_FIELDS))
    off = np.ascontiguousarray(batch.user_off, np.int64)
    bk = None if bucket is None else np.ascontiguousarray(bucket, np.int32)
    E = np.ascontiguousarray(res["E"], np.float64)
    El = np.ascontiguousarray(res["E_lc"], np.float64)
    nt = np.ascontiguousarray(res["n_tilde"], np.int32)
    fe = np.ascontiguousarray(res["f_e"], np.float64)
    ss = np.ascontiguousarray(res["status"], np.int32)
    lib().oracle_stats(n, off.ctypes.data_as(C.POINTER(C.c_longlong)), None if bk is None else _ip(bk), n_buckets,
                       _dp(E), _dp(El), _ip(nt), _dp(fe), _ip(ss), _dp(st))
    return st


def partition_from_plan(batch, res) -> np.ndarray:
    """Per-user partition points of a J-DOB plan: n~* for offloaders, N for locals."""
    part = np.zeros(batch.n_users, np.int32)
    for i in range(batch.n_inst):
        N = batch.models[batch.model_id[i]].N
        o0 = int(batch.user_off[i])
        for u in range(batch.M(i)):
            part[o0 + u] = res["n_tilde"][i] if (int(res["mask"][i]) >> u) & 1 else N
    return part


def og(batch, i=0, mode=MODE_FULL) -> dict:
    """Outer grouping DP over deadline-sorted users with the inner J-DOB (reading R21)."""
    keep = _Keep()
    r = OOgResult()
    lib().oracle_og(C.byref(_omodel(batch.models[batch.model_id[i]], keep)), C.byref(_oinst(batch, i, keep)),
                    mode, C.byref(r))
    M = batch.M(i)
    ng = r.n_groups
    return dict(E=r.E, t_free_next=r.t_free_next, status=r.status, n_groups=ng,
                group_of=np.array(r.group_of[:M]), part=np.array(r.part[:M]), f_user=np.array(r.f_user[:M]),
                group_fe=np.array(r.group_fe[:ng]), group_start=np.array(r.group_start[:ng + 1]))


def og_batch(batch, mode=MODE_FULL) -> dict:
    n = batch.n_inst
    rs = [og(batch, i, mode) for i in range(n)]
    out = dict(E=np.array([r["E"] for r in rs]), t_free_next=np.array([r["t_free_next"] for r in rs]),
               status=np.array([r["status"] for r in rs], np.int32),
               n_groups=np.array([r["n_groups"] for r in rs], np.int32),
               group_of=np.concatenate([r["group_of"] for r in rs]).astype(np.int32),
               part=np.concatenate([r["part"] for r in rs]).astype(np.int32),
               f_user=np.concatenate([r["f_user"] for r in rs]),
               group_fe=np.stack([np.pad(r["group_fe"], (0, 32 - len(r["group_fe"]))) for r in rs]))
    return out
