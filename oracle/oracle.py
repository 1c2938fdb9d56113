"""ctypes wrapper around the CPU oracle (oracle/cm_oracle.c).

TEST INFRASTRUCTURE ONLY: imported by tests/, __graft_entry__.smoke() and bench.py's
cpu_baseline / --impl reference legs.  The product package never imports this module.
Argument marshalling only; every computation happens in cm_oracle.c, which cites the
paper passage each function follows.
"""
from __future__ import annotations

import ctypes as C
import os
import subprocess

import numpy as np

_HERE = os.path.dirname(os.path.abspath(__file__))
_SRC = os.path.join(_HERE, "cm_oracle.c")
_LIB = os.path.join(_HERE, "libcm_oracle.so")
_LIB_OMP = os.path.join(_HERE, "libcm_oracle_omp.so")   # all-core timing build (bench cpu_baseline)

F32, BF16 = 0, 1
CFLAGS = ["-O2", "-std=c11", "-ffp-contract=off", "-fno-fast-math", "-fPIC", "-shared", "-Wall",
          "-Wno-unknown-pragmas"]


def build(force: bool = False, omp: bool = False) -> str:
    """Compile the oracle with gcc (plain C, no FMA contraction, no fast-math).  omp=True:
    the same source with -fopenmp (sampled trajectories split over the host's cores; used
    only to time the oracle on every core)."""
    out = _LIB_OMP if omp else _LIB
    if force or not os.path.exists(out) or os.path.getmtime(out) < os.path.getmtime(_SRC):
        tmp = out + f".tmp{os.getpid()}"
        subprocess.check_call(["gcc", *CFLAGS, *(["-fopenmp"] if omp else []), "-o", tmp, _SRC, "-lm"])
        os.replace(tmp, out)
    return out


_libs = {}


def lib(omp: bool = False):
    if omp not in _libs:
        L = C.CDLL(build(omp=omp))
        i64p = np.ctypeslib.ndpointer(np.int64, flags="C")
        i32p = np.ctypeslib.ndpointer(np.int32, flags="C")
        f32p = np.ctypeslib.ndpointer(np.float32, flags="C")
        u8p = np.ctypeslib.ndpointer(np.uint8, flags="C")
        L.cmo_fp_env_ok.restype = C.c_int
        L.cmo_plan.restype = C.c_int64
        L.cmo_plan.argtypes = [i64p, C.c_int32, C.c_int64, C.c_int32, C.c_int32, i32p, i32p,
                               i64p, i64p, i64p, i64p, C.POINTER(C.c_int64)]
        L.cmo_splitmix64.restype = C.c_uint64
        L.cmo_splitmix64.argtypes = [C.c_uint64]
        L.cmo_gen_f32.restype = C.c_float
        L.cmo_gen_f32.argtypes = [C.c_uint64, C.c_uint64, C.c_uint64, C.c_uint64, C.c_int32]
        L.cmo_gen_bf16val.restype = C.c_float
        L.cmo_gen_bf16val.argtypes = [C.c_uint64, C.c_uint64, C.c_uint64, C.c_uint64, C.c_int32]
        L.cmo_gen_p0.restype = C.c_float
        L.cmo_gen_p0.argtypes = [C.c_uint64, C.c_uint64]
        L.cmo_fill_grads.restype = None
        L.cmo_fill_grads.argtypes = [C.c_uint64, C.c_int32, C.c_int64, C.c_int32, C.c_int32, C.c_int64,
                                     i64p, i64p, i64p, C.c_void_p]
        L.cmo_fill_p0.restype = None
        L.cmo_fill_p0.argtypes = [C.c_uint64, C.c_int64, i64p, i64p, i64p, f32p]
        L.cmo_reduce_f32.restype = None
        L.cmo_reduce_f32.argtypes = [C.c_int32, C.c_int64, C.POINTER(C.c_void_p), f32p]
        L.cmo_reduce_bf16.restype = None
        L.cmo_reduce_bf16.argtypes = [C.c_int32, C.c_int64, C.POINTER(C.c_void_p), C.c_void_p]
        L.cmo_f32_to_bf16_rne.restype = C.c_uint16
        L.cmo_f32_to_bf16_rne.argtypes = [C.c_float]
        L.cmo_scalars.restype = C.c_int
        L.cmo_scalars.argtypes = [C.c_int64, C.c_double, C.c_double, C.c_double, C.c_double,
                                  C.c_double, C.c_int32, f32p]
        L.cmo_adamw_f32.restype = None
        L.cmo_adamw_f32.argtypes = [C.c_int64, f32p, f32p, f32p, f32p, f32p]
        L.cmo_adamw_bf16.restype = None
        L.cmo_adamw_bf16.argtypes = [C.c_int64, C.c_void_p, f32p, f32p, f32p, f32p]
        L.cmo_iteration.restype = None
        L.cmo_iteration.argtypes = [C.c_int32, C.c_int64, C.c_int32, C.POINTER(C.c_void_p), f32p,
                                    C.c_void_p, C.c_void_p, C.c_void_p, C.c_void_p, C.c_void_p,
                                    C.c_void_p, C.c_void_p, C.c_void_p]
        L.cmo_run_sample.restype = None
        L.cmo_run_sample.argtypes = [C.c_uint64, C.c_int32, C.c_int32, C.c_int32, C.c_int64, C.c_int64,
                                     C.c_double, C.c_double, C.c_double, C.c_double, C.c_double,
                                     C.c_int64, i64p, u8p, f32p, f32p, f32p, f32p]
        L.cmo_sample_init.restype = None
        L.cmo_sample_init.argtypes = [C.c_uint64, C.c_int64, i64p, u8p, f32p, f32p, f32p, f32p]
        L.cmo_sample_iterate.restype = None
        L.cmo_sample_iterate.argtypes = L.cmo_run_sample.argtypes
        L.cmo_sgd_scalars.restype = C.c_int
        L.cmo_sgd_scalars.argtypes = [C.c_double, C.c_double, C.c_double, C.c_int32, f32p]
        L.cmo_sgd_f32.restype = None
        L.cmo_sgd_f32.argtypes = [C.c_int64, f32p, f32p, f32p, f32p]
        L.cmo_sgd_bf16.restype = None
        L.cmo_sgd_bf16.argtypes = [C.c_int64, C.c_void_p, f32p, f32p, f32p]
        L.cmo_run_sample_sgd.restype = None
        L.cmo_run_sample_sgd.argtypes = [C.c_uint64, C.c_int32, C.c_int32, C.c_int32, C.c_int64, C.c_int64,
                                         C.c_double, C.c_double, C.c_double, C.c_int64, i64p, u8p, f32p, f32p,
                                         f32p]
        L.cmo_consolidate.restype = C.c_int64
        L.cmo_consolidate.argtypes = [C.c_int32, i64p]
        L.cmo_threads.restype = C.c_int
        _libs[omp] = L
    return _libs[omp]


def threads(omp: bool = False) -> int:
    return int(lib(omp).cmo_threads())


class Plan:
    """Result of the oracle planner."""

    def __init__(self, numel, cap_bytes, elem_size, world_size):
        numel = np.ascontiguousarray(numel, dtype=np.int64)
        nt = len(numel)
        bf = np.zeros(max(nt, 1), np.int32)
        bc = np.zeros(max(nt, 1), np.int32)
        bo = np.zeros(max(nt, 1), np.int64)
        bp = np.zeros(max(nt, 1), np.int64)
        bu = np.zeros(max(nt, 1), np.int64)
        to = np.zeros(max(nt, 1), np.int64)
        tot = C.c_int64(0)
        nb = lib().cmo_plan(numel if nt else np.zeros(1, np.int64), nt, int(cap_bytes), int(elem_size),
                            int(world_size), bf, bc, bo, bp, bu, to, C.byref(tot))
        if nb < 0:
            raise ValueError("oracle planner rejected the layer table")
        self.n_buckets = int(nb)
        self.bucket_first = bf[:nb].copy()
        self.bucket_count = bc[:nb].copy()
        self.bucket_off = bo[:nb].copy()
        self.bucket_padded = bp[:nb].copy()
        self.bucket_used = bu[:nb].copy()
        self.tensor_off = to[:nt].copy()
        self.total = int(tot.value)
        self.world_size = int(world_size)
        self.elem_size = int(elem_size)

    def used_mask(self) -> np.ndarray:
        m = np.zeros(self.total, np.uint8)
        for o, u in zip(self.bucket_off, self.bucket_used):
            m[o:o + u] = 1
        return m


def scalars(step, lr=1e-3, b1=0.9, b2=0.999, eps=1e-8, wd=0.01, n=1) -> np.ndarray:
    out = np.zeros(10, np.float32)
    if lib().cmo_scalars(int(step), lr, b1, b2, eps, wd, int(n), out) != 0:
        raise ValueError("bad step / n")
    return out


def sgd_scalars(lr=1e-2, momentum=0.9, wd=0.0, n=1) -> np.ndarray:
    out = np.zeros(5, np.float32)
    if lib().cmo_sgd_scalars(lr, momentum, wd, int(n), out) != 0:
        raise ValueError("bad n")
    return out


def sgd(R, sc, p, buf, dtype=F32):
    """SGD with momentum (reading R27), in place on float32 p, buf."""
    if dtype == F32:
        lib().cmo_sgd_f32(len(p), np.ascontiguousarray(R, np.float32), sc, p, buf)
    else:
        R = np.ascontiguousarray(R, np.uint16)
        lib().cmo_sgd_bf16(len(p), R.ctypes.data, sc, p, buf)


def gen_grads(plan: Plan, seed, rank, t, dtype, s=10) -> np.ndarray:
    out = np.zeros(plan.total, np.float32 if dtype == F32 else np.uint16)
    lib().cmo_fill_grads(seed, rank, t, dtype, s, plan.n_buckets, plan.bucket_off, plan.bucket_padded,
                         plan.bucket_used, out.ctypes.data)
    return out


def gen_p0(plan: Plan, seed) -> np.ndarray:
    out = np.zeros(plan.total, np.float32)
    lib().cmo_fill_p0(seed, plan.n_buckets, plan.bucket_off, plan.bucket_padded, plan.bucket_used, out)
    return out


def _ptrs(arrs):
    return (C.c_void_p * len(arrs))(*[a.ctypes.data for a in arrs])


def reduce_f32(gs) -> np.ndarray:
    gs = [np.ascontiguousarray(g, np.float32) for g in gs]
    out = np.empty(len(gs[0]), np.float32)
    lib().cmo_reduce_f32(len(gs), len(gs[0]), _ptrs(gs), out)
    return out


def reduce_bf16(gs) -> np.ndarray:
    gs = [np.ascontiguousarray(g, np.uint16) for g in gs]
    out = np.empty(len(gs[0]), np.uint16)
    lib().cmo_reduce_bf16(len(gs), len(gs[0]), _ptrs(gs), out.ctypes.data)
    return out


def f32_to_bf16(x: float) -> int:
    return int(lib().cmo_f32_to_bf16_rne(float(x)))


def adamw(R, sc, p, m, v, dtype=F32):
    """In place on float32 arrays p, m, v."""
    if dtype == F32:
        lib().cmo_adamw_f32(len(p), np.ascontiguousarray(R, np.float32), sc, p, m, v)
    else:
        R = np.ascontiguousarray(R, np.uint16)
        lib().cmo_adamw_bf16(len(p), R.ctypes.data, sc, p, m, v)


class Run:
    """Whole-buffer oracle run of the path: per-rank grads -> R (rank-order sum) ->
    tap T -> trainer AdamW and an independent shadow AdamW.
    opt="sgd": the same path with SGD-momentum (hp keys lr, momentum, wd; the velocity
    lives in m, v stays zero)."""

    def __init__(self, plan: Plan, seed=0, dtype=F32, gscale=10, hp=None, shadow=True, opt="adamw"):
        self.plan, self.seed, self.dtype, self.gscale = plan, seed, dtype, gscale
        self.opt = opt
        if opt == "sgd":
            self.hp = dict(lr=1e-2, momentum=0.9, wd=0.0)
        else:
            self.hp = dict(lr=1e-3, b1=0.9, b2=0.999, eps=1e-8, wd=0.01)
        if hp:
            self.hp.update(hp)
        n = plan.total
        self.p = gen_p0(plan, seed)
        self.m = np.zeros(n, np.float32)
        self.v = np.zeros(n, np.float32)
        self.shadow = shadow
        if shadow:
            self.sp, self.sm, self.sv = self.p.copy(), self.m.copy(), self.v.copy()
        self.t = 0
        gd = np.float32 if dtype == F32 else np.uint16
        self.R = np.zeros(n, gd)
        self.T = np.zeros(n, gd)

    def step(self, grads=None):
        """One iteration t -> t+1.  grads: list of per-rank flat buffers (else generated)."""
        n = self.plan.world_size
        if grads is None:
            grads = [gen_grads(self.plan, self.seed, r, self.t, self.dtype, self.gscale) for r in range(n)]
        if self.opt == "sgd":
            self.R[:] = reduce_f32(grads) if self.dtype == F32 else reduce_bf16(grads)
            self.T[:] = self.R                                   # tap: exactly R, once
            sc = sgd_scalars(n=n, **self.hp)
            sgd(self.R, sc, self.p, self.m, self.dtype)
            if self.shadow:
                sgd(self.T, sc, self.sp, self.sm, self.dtype)
            self.t += 1
            return grads
        sc = scalars(self.t + 1, n=n, **self.hp)
        null = None
        lib().cmo_iteration(n, self.plan.total, self.dtype, _ptrs(grads), sc, self.R.ctypes.data,
                            self.T.ctypes.data, self.p.ctypes.data, self.m.ctypes.data, self.v.ctypes.data,
                            self.sp.ctypes.data if self.shadow else null,
                            self.sm.ctypes.data if self.shadow else null,
                            self.sv.ctypes.data if self.shadow else null)
        self.t += 1
        return grads


def run_sample(seed, n, dtype, gscale, steps, idx, used, t0=0, lr=1e-3, b1=0.9, b2=0.999, eps=1e-8, wd=0.01,
               omp=False):
    """Trajectory of sampled flat indices over `steps` iterations.
    omp=True runs the all-core build (same arithmetic per element)."""
    idx = np.ascontiguousarray(idx, np.int64)
    used = np.ascontiguousarray(used, np.uint8)
    k = len(idx)
    p, m, v, R = (np.zeros(k, np.float32) for _ in range(4))
    lib(omp).cmo_run_sample(seed, n, dtype, gscale, t0, steps, lr, b1, b2, eps, wd, k, idx, used, p, m, v, R)
    return p, m, v, R


class SampleRun:
    """Sampled trajectories advanced one call at a time (state held here): bench.py times
    single oracle iterations with it.  Same arithmetic as run_sample."""

    def __init__(self, seed, n, dtype, gscale, idx, used, lr=1e-3, b1=0.9, b2=0.999, eps=1e-8, wd=0.01,
                 omp=False):
        self.idx = np.ascontiguousarray(idx, np.int64)
        self.used = np.ascontiguousarray(used, np.uint8)
        k = len(self.idx)
        self.p, self.m, self.v, self.R = (np.zeros(k, np.float32) for _ in range(4))
        self.args = (seed, n, dtype, gscale)
        self.hp = (lr, b1, b2, eps, wd)
        self.L = lib(omp)
        self.t = 0
        self.L.cmo_sample_init(seed, k, self.idx, self.used, self.p, self.m, self.v, self.R)

    def iterate(self, steps=1):
        self.L.cmo_sample_iterate(*self.args, self.t, steps, *self.hp, len(self.idx), self.idx, self.used,
                                  self.p, self.m, self.v, self.R)
        self.t += steps


def run_sample_sgd(seed, n, dtype, gscale, steps, idx, used, t0=0, lr=1e-2, momentum=0.9, wd=0.0):
    """SGD-momentum trajectory of sampled flat indices -> (p, buf, R_last)."""
    idx = np.ascontiguousarray(idx, np.int64)
    used = np.ascontiguousarray(used, np.uint8)
    k = len(idx)
    p, b, R = (np.zeros(k, np.float32) for _ in range(3))
    lib().cmo_run_sample_sgd(seed, n, dtype, gscale, t0, steps, lr, momentum, wd, k, idx, used, p, b, R)
    return p, b, R


def consolidate(last_steps) -> int:
    a = np.ascontiguousarray(last_steps, np.int64)
    return int(lib().cmo_consolidate(len(a), a))
