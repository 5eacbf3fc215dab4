"""Thin ctypes binding over libjdob.so (include/jdob.h).

Argument marshalling only: every step of the hot path runs in the CUDA kernels of
libjdob.so.  PyTorch provides device memory and streams.  There is no CPU fallback:
if the library is missing or no CUDA device is present, calls raise.
"""
from __future__ import annotations

import ctypes as C
import os
import threading
from typing import Optional

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.environ.get("JDOB_LIB") or os.path.join(HERE, "libjdob.so")

MAX_M, MAX_N, MAX_K, STATS_FIELDS, MAX_BUCKETS = 32, 63, 65536, 80, 64
OK, EINVAL, ETOOBIG, ECUDA = 0, 1, 2, 3
ST_OK, ST_LOCAL_INFEASIBLE, ST_REQUIRE, ST_BADPARAM, ST_BADMODEL, ST_TOOBIG = range(6)
MODE_FULL, MODE_LC, MODE_NO_EDGE_DVFS, MODE_BINARY = range(4)
SPACE_GENERAL, SPACE_IDENTICAL = 0, 1

_P = C.POINTER
_D = _P(C.c_double)


class JModel(C.Structure):
    _fields_ = [("N", C.c_int32), ("B_max", C.c_int32)] + [(f, C.c_void_p) for f in ("A", "O", "g", "q", "d", "c")]


class JBatch(C.Structure):
    _fields_ = [("n_inst", C.c_int64), ("n_models", C.c_int32), ("model_id", C.c_void_p), ("user_off", C.c_void_p)] + \
               [(f, C.c_void_p) for f in ("zeta", "kappa", "f_min", "f_max", "R", "p_u", "T",
                                          "t_free", "fe_min", "fe_max", "rho", "bucket")]


class JResult(C.Structure):
    _fields_ = [(f, C.c_void_p) for f in ("E", "E_lc", "t_free_next", "f_e", "n_tilde", "j", "status", "mask",
                                          "f_user", "counts", "stats")] + [("n_buckets", C.c_int32),
                                                                           ("partition", C.c_void_p),
                                                                           ("work", C.c_void_p),
                                                                           ("violations", C.c_void_p),
                                                                           ("slack", C.c_double)]


class JGenParams(C.Structure):
    _fields_ = [("seed", C.c_uint64), ("inst_begin", C.c_int64), ("hetero", C.c_int32)] + \
               [(f, C.c_double) for f in ("zeta", "kappa", "f_min", "f_max", "R", "p_u", "fe_min", "fe_max")] + \
               [("rho", C.c_double * 3), ("lat", C.c_double * 3)]


class JSharedBatch(C.Structure):
    _fields_ = [("n_inst", C.c_int64), ("n_models", C.c_int32), ("model_id", C.c_void_p), ("user_off", C.c_void_p)] + \
               [(f, C.c_void_p) for f in ("zeta", "kappa", "f_min", "f_max", "R", "p_u", "T",
                                          "t_free", "fe_min", "fe_max", "rho", "bucket")]


class JGrouped(C.Structure):
    _fields_ = [(f, C.c_void_p) for f in ("E", "t_free_next", "n_groups", "status", "group_of", "partition", "f_user",
                                          "group_fe")]


_lock = threading.Lock()
_lib = None


class JdobError(RuntimeError):
    pass


def _sig(L, name, argtypes, restype=None):
    """Declare a C-ABI signature.  A library chosen by JDOB_LIB (an older build for an A/B timing) may
    lack entry points added later: those are skipped there; the in-tree library must export all."""
    if not hasattr(L, name):
        if os.environ.get("JDOB_LIB"):
            return
        raise ImportError(f"{LIB_PATH} does not export {name}")
    f = getattr(L, name)
    f.argtypes = argtypes
    if restype is not None:
        f.restype = restype


def lib():
    """Load libjdob.so (built in-tree by paper_2504_14611_b200.build)."""
    global _lib
    with _lock:
        if _lib is None:
            if not os.path.exists(LIB_PATH):
                raise ImportError(f"libjdob.so not built ({LIB_PATH}); run __graft_entry__.build() "
                                  "or python -m paper_2504_14611_b200.build")
            L = C.CDLL(LIB_PATH)
            _sig(L, "jdob_workspace_bytes", [_P(JModel), C.c_int32, C.c_int32], C.c_size_t)
            _sig(L, "jdob_solve_batch", [_P(JModel), C.c_int32, _P(JBatch), C.c_int32, _P(JResult), C.c_void_p, C.c_size_t, C.c_void_p])
            _sig(L, "jdob_solve_batch_modes", [_P(JModel), C.c_int32, _P(JBatch), _P(JResult), C.c_void_p, C.c_size_t,
                                               C.c_void_p])
            _sig(L, "jdob_solve_batch_host", [_P(JModel), C.c_int32, _P(JBatch), C.c_int32, _P(JResult), C.c_void_p, _P(C.c_int64), _P(C.c_int64)])
            _sig(L, "jdob_bruteforce", [_P(JModel), C.c_int32, _P(JBatch), C.c_int32, C.c_uint64, C.c_uint64, C.c_void_p, C.c_void_p, C.c_void_p, C.c_void_p, C.c_void_p, C.c_size_t, C.c_void_p])
            _sig(L, "jdob_stats", [_P(JBatch), _P(JResult), C.c_void_p, C.c_size_t, C.c_void_p])
            _sig(L, "jdob_stats_part", [_P(JBatch), _P(JResult), C.c_int64, C.c_int32, C.c_int32, C.c_void_p, C.c_size_t, C.c_void_p])
            _sig(L, "jdob_bf_space_size", [C.c_int32, C.c_int32, C.c_int32, C.c_int64], C.c_uint64)
            _sig(L, "jdob_eval", [_P(JModel), C.c_int32, _P(JBatch), C.c_void_p, C.c_void_p, C.c_void_p, C.c_void_p, C.c_double, C.c_void_p, C.c_void_p, C.c_void_p, C.c_void_p, C.c_void_p, C.c_void_p, C.c_size_t, C.c_void_p])
            _sig(L, "jdob_grouped_workspace_bytes", [_P(JModel), C.c_int32, C.c_int64, C.c_int64], C.c_size_t)
            _sig(L, "jdob_solve_grouped", [_P(JModel), C.c_int32, _P(JBatch), C.c_int32, _P(JGrouped), C.c_void_p, C.c_size_t, C.c_void_p])
            _sig(L, "jdob_solve_shared_host", [_P(JModel), C.c_int32, _P(JSharedBatch), C.c_int32, _P(JResult),
                                               C.c_void_p, _P(C.c_int64), _P(C.c_int64)])
            _sig(L, "jdob_generate_workspace_bytes", [C.c_int64], C.c_size_t)
            _sig(L, "jdob_generate_c5_instances", [_P(JGenParams), _P(JBatch), _P(C.c_int64), C.c_void_p, C.c_size_t, C.c_void_p])
            _sig(L, "jdob_generate_c5_users", [_P(JGenParams), _P(JBatch), C.c_void_p, C.c_size_t, C.c_void_p])
            L.jdob_last_error.restype = C.c_char_p
            L.jdob_version.restype = C.c_char_p
            L.jdob_release_pool.restype = C.c_int
            _lib = L
    return _lib


EXPORTED = ("jdob_workspace_bytes", "jdob_solve_batch", "jdob_solve_batch_host", "jdob_bruteforce",
            "jdob_bf_space_size", "jdob_eval", "jdob_grouped_workspace_bytes", "jdob_solve_grouped",
            "jdob_last_error", "jdob_version", "jdob_release_pool", "jdob_stats", "jdob_stats_part",
            "jdob_generate_workspace_bytes", "jdob_generate_c5_instances", "jdob_generate_c5_users",
            "jdob_solve_shared_host", "jdob_solve_batch_modes")


def _check(rc):
    if rc != OK:
        raise JdobError(f"jdob error {rc}: {lib().jdob_last_error().decode()}")


def _torch():
    import torch
    if not torch.cuda.is_available():
        raise RuntimeError("paper_2504_14611_b200 needs a CUDA device (B200, sm_100a); there is no CPU path")
    return torch


def _ptr(t) -> Optional[int]:
    return None if t is None else t.data_ptr()


def _stream_handle(stream) -> Optional[int]:
    torch = _torch()
    if stream is None:
        stream = torch.cuda.current_stream()
    return stream.cuda_stream


class DeviceBatch:
    """A batch resident in device memory (torch tensors) plus its C-ABI descriptors.

    `batch` is any object with the fields of include/jdob.h's jdob_batch (numpy
    arrays): models (list with N, B_max, A, O, g, q, d, c), model_id, user_off, zeta,
    kappa, f_min, f_max, R, p_u, T, t_free, fe_min, fe_max, rho, optional bucket.
    """

    USER = ("zeta", "kappa", "f_min", "f_max", "R", "p_u", "T")
    INST = ("t_free", "fe_min", "fe_max", "rho")

    def __init__(self, batch, device=None, non_blocking=False):
        torch = _torch()
        self.device = torch.device(device if device is not None else "cuda")
        dev = self.device

        def up(a, dtype):
            t = torch.from_numpy(np.ascontiguousarray(a)).to(dtype)
            return t.to(dev, non_blocking=non_blocking)

        self._set_models(batch.models, up)
        self.n_inst = int(len(batch.model_id))
        self.user_off_host = np.ascontiguousarray(batch.user_off, np.int64)
        self.n_users = int(self.user_off_host[-1])
        self.t = {"model_id": up(batch.model_id, torch.int32), "user_off": up(self.user_off_host, torch.int64)}
        for f in self.USER + self.INST:
            self.t[f] = up(np.asarray(getattr(batch, f), np.float64), torch.float64)
        bucket = getattr(batch, "bucket", None)
        self.t["bucket"] = None if bucket is None else up(bucket, torch.int32)
        self.n_buckets = int(getattr(batch, "meta", {}).get("n_buckets", MAX_M)) if bucket is not None else MAX_M
        self.jbatch = JBatch(self.n_inst, self.n_models, *[_ptr(self.t[f]) for f in
                                                           ("model_id", "user_off") + self.USER + self.INST +
                                                           ("bucket",)])
        self._ws = {}

    def _set_models(self, models, up):
        torch = _torch()
        self.model_tensors = []
        ms = []
        for m in models:
            mt = {f: up(np.asarray(getattr(m, f), np.float64), torch.float64) for f in ("A", "O", "g", "q", "d", "c")}
            self.model_tensors.append(mt)
            ms.append(JModel(int(m.N), int(m.B_max), *[mt[f].data_ptr() for f in ("A", "O", "g", "q", "d", "c")]))
        self.Ns = [int(m.N) for m in models]
        self.n_models = len(ms)
        self.jmodels = (JModel * len(ms))(*ms)

    @classmethod
    def generate_c5(cls, models, params: dict, n_inst: int, device=None, n_buckets: int = 480, stream=None):
        """The C5 workload generated on the device (jdob_generate_c5_*; input plumbing, bit-identical
        to jdobgen.config_c5): `models` and `params` (the jdob_gen_params fields) come from the caller,
        e.g. jdobgen.c5_device_inputs.  No host->device traffic but the model tables."""
        torch = _torch()
        self = cls.__new__(cls)
        self.device = torch.device(device if device is not None else "cuda")
        dev = self.device

        def up(a, dtype):
            return torch.from_numpy(np.ascontiguousarray(a)).to(dtype).to(dev)

        self._set_models(models, up)
        n = int(n_inst)
        self.n_inst = n
        gp = JGenParams(int(params["seed"]), int(params.get("inst_begin", 0)), int(params.get("hetero", 0)),
                        *[float(params[f]) for f in ("zeta", "kappa", "f_min", "f_max", "R", "p_u", "fe_min",
                                                      "fe_max")],
                        (C.c_double * 3)(*params["rho"]), (C.c_double * 3)(*params["lat"]))
        self.t = {"model_id": torch.empty(n, dtype=torch.int32, device=dev),
                  "user_off": torch.empty(n + 1, dtype=torch.int64, device=dev),
                  "bucket": torch.empty(n, dtype=torch.int32, device=dev)}
        for f in self.INST:
            self.t[f] = torch.empty(n, dtype=torch.float64, device=dev)
        for f in self.USER:
            self.t[f] = None
        ws = torch.empty(int(lib().jdob_generate_workspace_bytes(n)), dtype=torch.uint8, device=dev)
        jb = JBatch(n, self.n_models, *[_ptr(self.t[f]) for f in ("model_id", "user_off") + self.USER + self.INST +
                                        ("bucket",)])
        nu = C.c_int64()
        sh = _stream_handle(stream)
        _check(lib().jdob_generate_c5_instances(C.byref(gp), C.byref(jb), C.byref(nu), ws.data_ptr(), ws.numel(), sh))
        self.n_users = int(nu.value)
        for f in self.USER:
            self.t[f] = torch.empty(self.n_users, dtype=torch.float64, device=dev)
        self.jbatch = JBatch(n, self.n_models, *[_ptr(self.t[f]) for f in
                                                 ("model_id", "user_off") + self.USER + self.INST + ("bucket",)])
        _check(lib().jdob_generate_c5_users(C.byref(gp), C.byref(self.jbatch), ws.data_ptr(), ws.numel(), sh))
        self.user_off_host = None
        self.n_buckets = n_buckets
        self._ws = {}
        return self

    def workspace(self, which: int):
        torch = _torch()
        if which not in self._ws:
            nb = lib().jdob_workspace_bytes(self.jmodels, self.n_models, which)
            if nb == 0:
                raise JdobError("jdob_workspace_bytes returned 0")
            self._ws[which] = torch.empty(int(nb), dtype=torch.uint8, device=self.device)
        return self._ws[which]


def solve_batch(db: DeviceBatch, mode: int = MODE_FULL, f_user: bool = True, counts: bool = False,
                stats: bool = False, n_buckets: Optional[int] = None, stream=None, out: Optional[dict] = None,
                partition: bool = False, work: bool = False, verify: bool = False, slack: float = 1e-9) -> dict:
    """jdob_solve_batch: J-DOB (Alg. 1/2) over every instance of `db`; outputs are device tensors.
    verify: the plans re-verified in the solver's epilogue with jdob_eval's formulas (row a11) ->
    out["violations"] (uint32 bits as int32), the bits jdob_eval returns for the same plans."""
    torch = _torch()
    dev = db.device
    n, nu = db.n_inst, db.n_users
    if out is None:
        out = dict(E=torch.empty(n, dtype=torch.float64, device=dev),
                   E_lc=torch.empty(n, dtype=torch.float64, device=dev),
                   t_free_next=torch.empty(n, dtype=torch.float64, device=dev),
                   f_e=torch.empty(n, dtype=torch.float64, device=dev),
                   n_tilde=torch.empty(n, dtype=torch.int32, device=dev),
                   j=torch.empty(n, dtype=torch.int32, device=dev),
                   status=torch.empty(n, dtype=torch.int32, device=dev),
                   mask=torch.empty(n, dtype=torch.int32, device=dev))
        if f_user:
            out["f_user"] = torch.empty(nu, dtype=torch.float64, device=dev)
        if counts:
            out["counts"] = torch.empty((n, 3), dtype=torch.int64, device=dev)
        if stats:
            nb = n_buckets if n_buckets is not None else db.n_buckets
            out["stats"] = torch.empty((nb, STATS_FIELDS), dtype=torch.float64, device=dev)
        if partition:
            out["partition"] = torch.empty(nu, dtype=torch.int32, device=dev)
        if work:
            out["work"] = torch.empty((n, 4), dtype=torch.int64, device=dev)
        if verify:
            out["violations"] = torch.empty(n, dtype=torch.int32, device=dev)
    r = JResult(*[_ptr(out.get(f)) for f in ("E", "E_lc", "t_free_next", "f_e", "n_tilde", "j", "status", "mask",
                                             "f_user", "counts", "stats")],
                int(out["stats"].shape[0]) if out.get("stats") is not None else 0, _ptr(out.get("partition")),
                _ptr(out.get("work")), _ptr(out.get("violations")), float(slack))
    ws = db.workspace(0)
    _check(lib().jdob_solve_batch(db.jmodels, db.n_models, C.byref(db.jbatch), int(mode), C.byref(r),
                                  ws.data_ptr(), ws.numel(), _stream_handle(stream)))
    return out


def solve_batch_modes(db: DeviceBatch, f_user: bool = True, stats: bool = False, n_buckets: Optional[int] = None,
                      partition: bool = False, stream=None) -> dict:
    """jdob_solve_batch_modes: J-DOB, J-DOB without edge DVFS and binary J-DOB (NEXT-2) in one pass;
    returns {MODE_FULL: res, MODE_NO_EDGE_DVFS: res, MODE_BINARY: res}, each as solve_batch's dict."""
    torch = _torch()
    dev = db.device
    n, nu = db.n_inst, db.n_users
    outs, rs = {}, []
    for mode in (MODE_FULL, MODE_NO_EDGE_DVFS, MODE_BINARY):
        o = dict(E=torch.empty(n, dtype=torch.float64, device=dev),
                 E_lc=torch.empty(n, dtype=torch.float64, device=dev),
                 t_free_next=torch.empty(n, dtype=torch.float64, device=dev),
                 f_e=torch.empty(n, dtype=torch.float64, device=dev),
                 n_tilde=torch.empty(n, dtype=torch.int32, device=dev),
                 j=torch.empty(n, dtype=torch.int32, device=dev),
                 status=torch.empty(n, dtype=torch.int32, device=dev),
                 mask=torch.empty(n, dtype=torch.int32, device=dev))
        if f_user:
            o["f_user"] = torch.empty(nu, dtype=torch.float64, device=dev)
        if stats:
            nb = n_buckets if n_buckets is not None else db.n_buckets
            o["stats"] = torch.empty((nb, STATS_FIELDS), dtype=torch.float64, device=dev)
        if partition:
            o["partition"] = torch.empty(nu, dtype=torch.int32, device=dev)
        outs[mode] = o
        rs.append(JResult(*[_ptr(o.get(f)) for f in ("E", "E_lc", "t_free_next", "f_e", "n_tilde", "j", "status",
                                                     "mask", "f_user")], None, _ptr(o.get("stats")),
                          int(o["stats"].shape[0]) if o.get("stats") is not None else 0, _ptr(o.get("partition")),
                          None, None, 0.0))
    arr = (JResult * 3)(*rs)
    ws = db.workspace(0)
    _check(lib().jdob_solve_batch_modes(db.jmodels, db.n_models, C.byref(db.jbatch), arr, ws.data_ptr(), ws.numel(),
                                        _stream_handle(stream)))
    return outs


def stats(db: DeviceBatch, res: dict, n_buckets: Optional[int] = None, stream=None, out=None,
          part: Optional[tuple] = None):
    """jdob_stats: the bucketed energy-saving statistics (a12) of solved instances `res` (the dict
    solve_batch returned for `db`), as a call of its own; returns the [n_buckets, 80] f64 tensor.
    part = (n_total, parts, p): `db` is part p of `parts` of a batch of n_total instances
    (jdob_stats_part); the result is that part's subtree root, folded by dist.fold_stats."""
    torch = _torch()
    if out is None:
        nb = n_buckets if n_buckets is not None else db.n_buckets
        out = torch.empty((nb, STATS_FIELDS), dtype=torch.float64, device=db.device)
    r = JResult(*[_ptr(res.get(f)) for f in ("E", "E_lc", "t_free_next", "f_e", "n_tilde", "j", "status", "mask")],
                None, None, out.data_ptr(), int(out.shape[0]), None, None)
    ws = db.workspace(2)
    if part is None:
        _check(lib().jdob_stats(C.byref(db.jbatch), C.byref(r), ws.data_ptr(), ws.numel(), _stream_handle(stream)))
    else:
        n_total, parts, p = part
        _check(lib().jdob_stats_part(C.byref(db.jbatch), C.byref(r), int(n_total), int(parts), int(p),
                                     ws.data_ptr(), ws.numel(), _stream_handle(stream)))
    return out


def eval_plans(db: DeviceBatch, partition=None, f_e=None, slack: float = 1e-9, f_user: bool = True,
               plans: Optional[dict] = None, stream=None, out: Optional[dict] = None) -> dict:
    """jdob_eval: D20-D22 (generalised, R14/R15) and violation bits for given configurations.

    Either `partition` (per-user n_m, device int32) with `f_e`, or `plans` = the dict
    returned by solve_batch (identical plans n_tilde/mask/f_e, re-verified in place)."""
    torch = _torch()
    dev = db.device
    n, nu = db.n_inst, db.n_users
    if plans is not None:
        part, nt, mk, fe = None, plans["n_tilde"], plans["mask"], plans["f_e"]
    else:
        part = partition.to(dev, torch.int32).contiguous()
        nt = mk = None
        fe = f_e.to(dev, torch.float64).contiguous()
    if out is None:
        out = dict(E=torch.empty(n, dtype=torch.float64, device=dev),
                   t_free_next=torch.empty(n, dtype=torch.float64, device=dev),
                   f_user=torch.empty(nu, dtype=torch.float64, device=dev) if f_user else None,
                   violations=torch.empty(n, dtype=torch.int32, device=dev),
                   status=torch.empty(n, dtype=torch.int32, device=dev))
    ws = db.workspace(0)
    _check(lib().jdob_eval(db.jmodels, db.n_models, C.byref(db.jbatch), _ptr(part), _ptr(nt), _ptr(mk),
                           fe.data_ptr(), float(slack), out["E"].data_ptr(), out["t_free_next"].data_ptr(),
                           _ptr(out["f_user"]), out["violations"].data_ptr(), out["status"].data_ptr(),
                           ws.data_ptr(), ws.numel(), _stream_handle(stream)))
    return out


def plan_partition(db: DeviceBatch, res: dict):
    """Per-user partition points of J-DOB plans (n~* for offloaders, N for locals): the kernel's own
    `partition` output, requested with solve_batch(..., partition=True)."""
    if res.get("partition") is None:
        raise ValueError("solve_batch(..., partition=True) writes the per-user partition")
    return res["partition"]


def release_pool() -> None:
    """jdob_release_pool: trim the device memory the host API's private pool keeps between calls."""
    _check(lib().jdob_release_pool())


def bf_space_size(space: int, N: int, M: int, k: int) -> int:
    return int(lib().jdob_bf_space_size(int(space), int(N), int(M), int(k)))


def bruteforce(db: DeviceBatch, space: int, idx_begin: int = 0, idx_end: Optional[int] = None, stream=None,
               work: bool = False):
    """jdob_bruteforce over [idx_begin, idx_end) of the single instance of `db`.

    Returns device tensors (E_min [1] f64, idx_min [1] i64, status [1] i32), plus the executed-work
    counters [9] i64 (include/jdob.h) when `work` is set."""
    torch = _torch()
    if db.n_inst != 1:
        raise ValueError("bruteforce needs a single-instance batch")
    if idx_end is None:
        idx_end = (1 << 64) - 1
    dev = db.device
    E = torch.empty(1, dtype=torch.float64, device=dev)
    I = torch.empty(1, dtype=torch.int64, device=dev)
    S = torch.empty(1, dtype=torch.int32, device=dev)
    W = torch.empty(9, dtype=torch.int64, device=dev) if work else None
    ws = db.workspace(1)
    _check(lib().jdob_bruteforce(db.jmodels, db.n_models, C.byref(db.jbatch), int(space), int(idx_begin),
                                 int(idx_end), E.data_ptr(), I.data_ptr(), S.data_ptr(), _ptr(W), ws.data_ptr(),
                                 ws.numel(), _stream_handle(stream)))
    return (E, I, S, W) if work else (E, I, S)


def shared_params(batch):
    """Per-instance (zeta, kappa, f_min, f_max, R, p_u) when every instance's users share them bit for bit
    (jdob_shared_batch), else None."""
    off = np.asarray(batch.user_off, np.int64)
    first = off[:-1]
    M = np.diff(off)
    if len(first) == 0 or (M < 1).any():
        return None
    out = {}
    for f in ("zeta", "kappa", "f_min", "f_max", "R", "p_u"):
        a = np.asarray(getattr(batch, f), np.float64)
        v = a[first]
        if not np.array_equal(a.view(np.int64), np.repeat(v, M).view(np.int64)):
            return None
        out[f] = v
    return out


class HostBuffers:
    """Pinned host copies of a batch and its outputs for the end-to-end call.  shared=True stores the
    users' device parameters once per instance (jdob_shared_batch; the batch's users must share them)."""

    def __init__(self, batch, f_user=False, stats=False, n_buckets=None, partition=False, shared=False):
        torch = _torch()

        def pin(a, dtype):
            t = torch.from_numpy(np.ascontiguousarray(a).astype(dtype, copy=False)).pin_memory()
            return t

        self.models = [{f: pin(np.asarray(getattr(m, f), np.float64), np.float64) for f in ("A", "O", "g", "q", "d", "c")}
                       for m in batch.models]
        self.jmodels = (JModel * len(self.models))(*[
            JModel(int(m.N), int(m.B_max), *[mt[f].data_ptr() for f in ("A", "O", "g", "q", "d", "c")])
            for m, mt in zip(batch.models, self.models)])
        self.n_models = len(self.models)
        n = len(batch.model_id)
        self.n_inst = n
        self.t = {"model_id": pin(batch.model_id, np.int32), "user_off": pin(batch.user_off, np.int64)}
        self.shared = bool(shared)
        sp = shared_params(batch) if shared else None
        if shared and sp is None:
            raise ValueError("shared=True needs users that share their parameters within each instance")
        for f in DeviceBatch.USER + DeviceBatch.INST:
            self.t[f] = pin(sp[f] if (sp is not None and f in sp) else getattr(batch, f), np.float64)
        bucket = getattr(batch, "bucket", None)
        self.t["bucket"] = None if bucket is None else pin(bucket, np.int32)
        cls = JSharedBatch if shared else JBatch
        self.jbatch = cls(n, self.n_models, *[_ptr(self.t[f]) for f in
                                               ("model_id", "user_off") + DeviceBatch.USER + DeviceBatch.INST +
                                               ("bucket",)])
        nu = int(batch.user_off[-1])
        z = lambda k, dt: torch.empty(k, dtype=dt).pin_memory()
        self.out = dict(E=z(n, torch.float64), E_lc=z(n, torch.float64), t_free_next=z(n, torch.float64),
                        f_e=z(n, torch.float64), n_tilde=z(n, torch.int32), j=z(n, torch.int32),
                        status=z(n, torch.int32), mask=z(n, torch.int32),
                        f_user=z(nu, torch.float64) if f_user else None, counts=None,
                        partition=z(nu, torch.int32) if partition else None,
                        stats=z((n_buckets or MAX_M) * STATS_FIELDS, torch.float64) if stats else None)
        self.n_buckets = (n_buckets or MAX_M) if stats else 0


def solve_batch_host(hb: HostBuffers, mode: int = MODE_FULL, stream=None):
    """jdob_solve_batch_host (jdob_solve_shared_host for shared HostBuffers): host buffers in, host buffers
    out (copies inside the call).

    Returns (h2d_bytes, d2h_bytes)."""
    o = hb.out
    r = JResult(*[_ptr(o.get(f)) for f in ("E", "E_lc", "t_free_next", "f_e", "n_tilde", "j", "status", "mask",
                                           "f_user", "counts", "stats")], hb.n_buckets, _ptr(o.get("partition")), None)
    h2d = C.c_int64()
    d2h = C.c_int64()
    fn = lib().jdob_solve_shared_host if hb.shared else lib().jdob_solve_batch_host
    _check(fn(hb.jmodels, hb.n_models, C.byref(hb.jbatch), int(mode), C.byref(r), _stream_handle(stream),
              C.byref(h2d), C.byref(d2h)))
    return h2d.value, d2h.value


def solve_grouped(db: DeviceBatch, mode: int = MODE_FULL, f_user: bool = True, stream=None) -> dict:
    """jdob_solve_grouped: outer grouping DP over deadline-sorted users with J-DOB inside (NEXT-1)."""
    torch = _torch()
    dev = db.device
    n, nu = db.n_inst, db.n_users
    out = dict(E=torch.empty(n, dtype=torch.float64, device=dev),
               t_free_next=torch.empty(n, dtype=torch.float64, device=dev),
               n_groups=torch.empty(n, dtype=torch.int32, device=dev),
               status=torch.empty(n, dtype=torch.int32, device=dev),
               group_of=torch.empty(nu, dtype=torch.int32, device=dev),
               partition=torch.empty(nu, dtype=torch.int32, device=dev),
               f_user=torch.empty(nu, dtype=torch.float64, device=dev) if f_user else None,
               group_fe=torch.empty((n, MAX_M), dtype=torch.float64, device=dev))
    nb = int(lib().jdob_grouped_workspace_bytes(db.jmodels, db.n_models, n, nu))
    if nb == 0:
        raise JdobError("jdob_grouped_workspace_bytes returned 0")
    key = ("grouped", nb)
    if key not in db._ws:
        db._ws[key] = torch.empty(nb, dtype=torch.uint8, device=dev)
    ws = db._ws[key]
    r = JGrouped(*[_ptr(out[f]) for f in ("E", "t_free_next", "n_groups", "status", "group_of", "partition",
                                          "f_user", "group_fe")])
    _check(lib().jdob_solve_grouped(db.jmodels, db.n_models, C.byref(db.jbatch), int(mode), C.byref(r),
                                    ws.data_ptr(), ws.numel(), _stream_handle(stream)))
    return out
