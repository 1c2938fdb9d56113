"""Thin ctypes binding of libcm.so (include/cm.h).  Argument marshalling only: every step
of the path runs in the library's sm_100a kernels.  Names mirror the C ABI.

There is no fallback: if libcm.so is missing or cannot load, importing a Context raises.
"""
from __future__ import annotations

import ctypes as C
import os

_HERE = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.path.join(_HERE, "libcm.so")

CM_OK, CM_ERR_ARG, CM_ERR_CONFIG, CM_ERR_INVARIANT, CM_ERR_UNRECOVERABLE, CM_ERR_CUDA, CM_ERR_STATE = range(7)
STATUS_NAMES = {0: "CM_OK", 1: "CM_ERR_ARG", 2: "CM_ERR_CONFIG", 3: "CM_ERR_INVARIANT",
                4: "CM_ERR_UNRECOVERABLE", 5: "CM_ERR_CUDA", 6: "CM_ERR_STATE"}
CM_F32, CM_BF16 = 0, 1
CM_VERIFY_SHADOW, CM_VERIFY_HOST, CM_VERIFY_RING = 1, 2, 4
CM_VERIFY_ALL = CM_VERIFY_SHADOW | CM_VERIFY_HOST | CM_VERIFY_RING
VERIFY_WHAT = {-1: None, 0: "p", 1: "m", 2: "v", 3: "ring", 4: "nonfinite", 5: "log_gap"}
CM_SHADOW_HOST, CM_SHADOW_DEVICE = 0, 1
CM_FLAG_NO_TAP = 1 << 0
CM_FLAG_ATTACH = 1 << 1
CM_FLAG_TAP_COPYENGINE = 1 << 2
CM_FLAG_NO_SHADOW = 1 << 3
CM_FLAG_ZERO1 = 1 << 5          # sharded AdamW state + fused parameter all-gather
CM_FLAG_TAP_DIRECT = 1 << 4     # default tap is "staged" (HBM staging + copy-engine drain)
CM_FLAG_NVLS = 1 << 6           # one-shot push through an NVLink-SHARP multicast inbox
CM_FLAG_OVERWRITE = 1 << 7      # replace a surviving shadow segment (else CM_ERR_STATE)

# every symbol include/cm.h declares (tests check the library exports all of them)
EXPORTS = ["cm_plan_buckets", "cm_plan_bucket_table", "cm_init", "cm_register_buckets", "cm_blob_size", "cm_connect",
           "cm_finalize", "cm_unlink_shadow", "cm_last_error", "cm_allreduce_multicast", "cm_apply_step", "cm_apply_bucket", "cm_apply_bucket_sgd",
           "cm_apply_step_sgd", "cm_shadow_apply", "cm_restore", "cm_gen_grads", "cm_init_state", "cm_verify", "cm_verify_ex", "cm_check", "cm_barrier", "cm_get_info",
           "cm_bucket_info", "cm_shadow_view", "cm_ring_view", "cm_timing", "cm_timing_bytes", "cm_set_param", "cm_join", "cm_shadow_save", "cm_shadow_load",
           "cm_crc32", "cm_shadow_query", "cm_shadow_consolidate", "cm_shadow_serve",
           "cm_shadow_export"]


class cm_shadow_desc(C.Structure):
    _fields_ = [("world_size", C.c_int32), ("rank", C.c_int32), ("dtype", C.c_int32), ("ring_depth", C.c_int32),
                ("n_buckets", C.c_int32), ("pad0", C.c_int32), ("shard_numel", C.c_int64),
                ("layout_hash", C.c_uint64), ("shadow_step", C.c_int64), ("half_step", C.c_int64 * 2),
                ("nf_step", C.c_int64)]


class cm_config(C.Structure):
    _fields_ = [("world_size", C.c_int32), ("rank", C.c_int32), ("device", C.c_int32),
                ("ring_depth", C.c_int32), ("shadow_place", C.c_int32), ("persist_every", C.c_int32),
                ("shm_name", C.c_char_p), ("flags", C.c_uint64)]


class cm_layer_table(C.Structure):
    _fields_ = [("numel", C.POINTER(C.c_int64)), ("n_tensors", C.c_int32), ("grad_dtype", C.c_int32),
                ("cap_bytes", C.c_int64)]


class cm_adamw(C.Structure):
    _fields_ = [("lr", C.c_double), ("beta1", C.c_double), ("beta2", C.c_double), ("eps", C.c_double),
                ("weight_decay", C.c_double)]


class cm_sgd(C.Structure):
    _fields_ = [("lr", C.c_double), ("momentum", C.c_double), ("weight_decay", C.c_double)]


class cm_info(C.Structure):
    _fields_ = [("n_buckets", C.c_int32), ("world_size", C.c_int32), ("rank", C.c_int32),
                ("ring_depth", C.c_int32), ("grad_dtype", C.c_int32), ("shadow_place", C.c_int32),
                ("peers_in_process", C.c_int32), ("drain_ctas", C.c_int32), ("numa_node", C.c_int32), ("padded_numel", C.c_int64),
                ("shard_numel", C.c_int64), ("shadow_step", C.c_int64), ("launches", C.c_int64),
                ("layout_hash", C.c_uint64), ("nonfinite_step", C.c_int64), ("nonfinite_index", C.c_int64),
                ("persist_every", C.c_int32), ("pad0", C.c_int32), ("host_half_step", C.c_int64 * 2)]


class CMError(RuntimeError):
    def __init__(self, status, msg):
        super().__init__(f"{STATUS_NAMES.get(status, status)}: {msg}")
        self.status = status


_lib = None


def lib():
    global _lib
    if _lib is None:
        if not os.path.exists(LIB_PATH):
            raise ImportError(f"{LIB_PATH} not built: run __graft_entry__.build()")
        L = C.CDLL(LIB_PATH)
        P = C.c_void_p
        L.cm_plan_buckets.argtypes = [C.POINTER(cm_layer_table), C.c_int32, C.POINTER(C.c_int64),
                                      C.POINTER(C.c_int32), C.POINTER(C.c_int64)]
        L.cm_plan_bucket_table.argtypes = [C.POINTER(cm_layer_table), C.c_int32, C.c_int32, C.POINTER(C.c_int64),
                                           C.POINTER(C.c_int64), C.POINTER(C.c_int64), C.POINTER(C.c_int32)]
        L.cm_init.argtypes = [C.POINTER(cm_config), C.POINTER(P)]
        L.cm_register_buckets.argtypes = [P, C.POINTER(cm_layer_table), P, P, P, P, P, C.POINTER(C.c_size_t)]
        L.cm_blob_size.restype = C.c_size_t
        L.cm_blob_size.argtypes = []
        L.cm_connect.argtypes = [P, P, C.c_size_t]
        L.cm_finalize.argtypes = [P]
        L.cm_unlink_shadow.argtypes = [C.c_char_p, C.c_int32]
        L.cm_last_error.restype = C.c_char_p
        L.cm_last_error.argtypes = [P]
        L.cm_allreduce_multicast.argtypes = [P, C.c_int32, C.c_int64, P]
        L.cm_apply_step.argtypes = [P, C.c_int64, C.POINTER(cm_adamw), P]
        L.cm_apply_step_sgd.argtypes = [P, C.c_int64, C.POINTER(cm_sgd), P]
        L.cm_apply_bucket.argtypes = [P, C.c_int32, C.c_int64, C.POINTER(cm_adamw), P]
        L.cm_apply_bucket_sgd.argtypes = [P, C.c_int32, C.c_int64, C.POINTER(cm_sgd), P]
        L.cm_shadow_apply.argtypes = [P, C.c_int64, P]
        L.cm_restore.argtypes = [P, C.POINTER(C.c_int64), P]
        L.cm_gen_grads.argtypes = [P, C.c_uint64, C.c_int64, C.c_int32, P]
        L.cm_init_state.argtypes = [P, C.c_uint64, P]
        L.cm_verify.argtypes = [P, C.POINTER(C.c_int64), P]
        L.cm_verify_ex.argtypes = [P, C.c_int32, C.POINTER(C.c_int64), C.POINTER(C.c_int32), P]
        L.cm_check.argtypes = [P, C.POINTER(C.c_int64), C.POINTER(C.c_int64)]
        L.cm_barrier.argtypes = [P, P]
        L.cm_get_info.argtypes = [P, C.POINTER(cm_info)]
        L.cm_bucket_info.argtypes = [P, C.c_int32, C.POINTER(C.c_int64), C.POINTER(C.c_int64), C.POINTER(C.c_int64)]
        L.cm_shadow_view.argtypes = [P, C.c_int32, C.POINTER(P), C.POINTER(P), C.POINTER(P)]
        L.cm_ring_view.argtypes = [P, C.c_int32, C.POINTER(P)]
        L.cm_set_param.argtypes = [P, C.c_char_p, C.c_int64]
        L.cm_join.argtypes = [P, P]
        L.cm_shadow_save.argtypes = [C.c_char_p, C.c_int32, C.c_char_p]
        L.cm_shadow_load.argtypes = [C.c_char_p, C.c_char_p, C.c_int32]
        L.cm_crc32.argtypes = [C.c_void_p, C.c_size_t]
        L.cm_shadow_query.argtypes = [C.c_char_p, C.c_int32, C.POINTER(cm_shadow_desc)]
        L.cm_shadow_consolidate.argtypes = [C.c_char_p, C.c_int32, C.POINTER(C.c_int64)]
        L.cm_shadow_serve.argtypes = [C.c_char_p, C.c_int32, C.c_int64, C.c_int32, C.c_int64, C.c_int64, C.c_void_p,
                                      C.POINTER(C.c_uint32)]
        L.cm_shadow_export.argtypes = [C.c_char_p, C.POINTER(cm_layer_table), C.c_int32, C.c_int64, C.c_char_p,
                                       C.POINTER(C.c_int64)]
        L.cm_timing.argtypes = [P, C.c_int32, C.POINTER(C.c_double), C.POINTER(C.c_int64)]
        L.cm_timing_bytes.argtypes = [P, C.POINTER(C.c_int64)]
        for name in EXPORTS:
            if name not in ("cm_blob_size", "cm_last_error", "cm_crc32"):
                getattr(L, name).restype = C.c_int     # cm_status
        L.cm_crc32.restype = C.c_uint32
        _lib = L
    return _lib


def _layer_table(numel, grad_dtype, cap_bytes):
    arr = (C.c_int64 * len(numel))(*[int(x) for x in numel])
    t = cm_layer_table(C.cast(arr, C.POINTER(C.c_int64)), len(numel), int(grad_dtype), int(cap_bytes))
    return t, arr


def plan_buckets(numel, grad_dtype, cap_bytes, world_size):
    """cm_plan_buckets -> (padded_numel, n_buckets, tensor_elem_offset list)."""
    t, keep = _layer_table(numel, grad_dtype, cap_bytes)
    tot = C.c_int64(0)
    nb = C.c_int32(0)
    offs = (C.c_int64 * max(len(numel), 1))()
    st = lib().cm_plan_buckets(C.byref(t), int(world_size), C.byref(tot), C.byref(nb), offs)
    if st != CM_OK:
        raise CMError(st, "cm_plan_buckets rejected the table")
    return tot.value, nb.value, list(offs[:len(numel)])


def plan_bucket_table(numel, grad_dtype, cap_bytes, world_size):
    """cm_plan_bucket_table -> list of (off, padded, used) per bucket (host-only)."""
    t, keep = _layer_table(numel, grad_dtype, cap_bytes)
    cap = max(len(numel), 1)
    off, pad, used = (C.c_int64 * cap)(), (C.c_int64 * cap)(), (C.c_int64 * cap)()
    nb = C.c_int32(0)
    st = lib().cm_plan_bucket_table(C.byref(t), int(world_size), cap, off, pad, used, C.byref(nb))
    if st != CM_OK:
        raise CMError(st, "cm_plan_bucket_table rejected the table")
    return [(off[b], pad[b], used[b]) for b in range(nb.value)]


def unlink_shadow(name, rank):
    return lib().cm_unlink_shadow(name.encode(), int(rank))


def shadow_save(name, rank, path):
    """Persist a rank's shadow segment to a CheckpointFile (CRC-32)."""
    st = lib().cm_shadow_save(name.encode(), int(rank), str(path).encode())
    if st != CM_OK:
        raise CMError(st, f"cm_shadow_save({name}, {rank}, {path})")


def shadow_load(path, name, rank):
    """Recreate a rank's shadow segment from a CheckpointFile (CRC-32 verified)."""
    st = lib().cm_shadow_load(str(path).encode(), name.encode(), int(rank))
    if st != CM_OK:
        raise CMError(st, f"cm_shadow_load({path}, {name}, {rank})")


def crc32(data) -> int:
    """cm_crc32 of bytes, or of a contiguous numpy array's memory (no copy)."""
    if isinstance(data, (bytes, bytearray)):
        return int(lib().cm_crc32(bytes(data), len(data)))
    assert data.flags.c_contiguous
    return int(lib().cm_crc32(data.ctypes.data if data.nbytes else None, data.nbytes))


def shadow_query(name, rank) -> "cm_shadow_desc":
    """cm_shadow_query: layout and snapshot-half steps of a rank's host segment."""
    d = cm_shadow_desc()
    st = lib().cm_shadow_query(name.encode(), int(rank), C.byref(d))
    if st != CM_OK:
        raise CMError(st, f"cm_shadow_query({name}, {rank})")
    return d


def shadow_consolidate(name, world_size) -> int:
    """cm_shadow_consolidate: the step I every shard can serve (min rule)."""
    i = C.c_int64(-1)
    st = lib().cm_shadow_consolidate(name.encode(), int(world_size), C.byref(i))
    if st != CM_OK:
        raise CMError(st, f"cm_shadow_consolidate({name}, {world_size})")
    return i.value


def shadow_serve(name, rank, step, what, off, count, out=None):
    """cm_shadow_serve into a host float32 array (allocated if out is None) -> (array, crc32)."""
    import numpy as np
    if out is None:
        out = np.empty(int(count), dtype=np.float32)
    assert out.dtype == np.float32 and out.flags.c_contiguous and out.size >= count
    crc = C.c_uint32(0)
    st = lib().cm_shadow_serve(name.encode(), int(rank), int(step), int(what), int(off), int(count),
                               out.ctypes.data if count else None, C.byref(crc))
    if st != CM_OK:
        raise CMError(st, f"cm_shadow_serve({name}, rank {rank}, step {step}, what {what}, [{off}, {off + count}))")
    return out, crc.value


def shadow_export(name, numel, grad_dtype, cap_bytes, world_size, path, step=-1) -> int:
    """cm_shadow_export: the checkpoint at `step` (default consolidated) as a per-tensor
    model file; returns the step written."""
    t, keep = _layer_table(numel, grad_dtype, cap_bytes)
    out = C.c_int64(-1)
    st = lib().cm_shadow_export(name.encode(), C.byref(t), int(world_size), int(step), str(path).encode(),
                                C.byref(out))
    if st != CM_OK:
        raise CMError(st, f"cm_shadow_export({name}, n={world_size}, step {step}, {path})")
    return out.value


def _stream_ptr(stream):
    if stream is None:
        return None
    if isinstance(stream, int):
        return stream
    return stream.cuda_stream   # torch.cuda.Stream


class Context:
    """One cm_ctx (one rank).  Methods mirror the C ABI one to one."""

    def __init__(self, world_size, rank, device, ring_depth=2, shadow_place=CM_SHADOW_HOST,
                 shm_name="checkmate", flags=0, persist_every=1):
        self._ctx = C.c_void_p()
        self._name = shm_name.encode() if shm_name else None
        cfg = cm_config(world_size, rank, device, ring_depth, shadow_place, persist_every, self._name, flags)
        st = lib().cm_init(C.byref(cfg), C.byref(self._ctx))
        if st != CM_OK:
            msg = self.last_error()
            self.finalize()
            raise CMError(st, msg)
        self._keep = []

    def last_error(self):
        if not self._ctx:
            return "no context"
        return lib().cm_last_error(self._ctx).decode(errors="replace")

    def _check(self, st):
        if st != CM_OK:
            raise CMError(st, self.last_error())

    def register_buckets(self, numel, grad_dtype, cap_bytes, grad_ptr, p_ptr, m_ptr, v_ptr) -> bytes:
        t, arr = _layer_table(numel, grad_dtype, cap_bytes)
        self._keep.append(arr)
        cap = lib().cm_blob_size()
        buf = C.create_string_buffer(cap)
        blen = C.c_size_t(cap)
        self._check(lib().cm_register_buckets(self._ctx, C.byref(t), grad_ptr, p_ptr, m_ptr, v_ptr, buf,
                                              C.byref(blen)))
        return buf.raw[:blen.value]

    def connect(self, blobs):
        data = b"".join(blobs)
        self._check(lib().cm_connect(self._ctx, data, len(blobs[0])))

    def allreduce_multicast(self, bucket, iteration, stream=None):
        self._check(lib().cm_allreduce_multicast(self._ctx, int(bucket), int(iteration), _stream_ptr(stream)))

    def apply_step(self, step, lr=1e-3, beta1=0.9, beta2=0.999, eps=1e-8, weight_decay=0.01, stream=None):
        hp = cm_adamw(lr, beta1, beta2, eps, weight_decay)
        self._check(lib().cm_apply_step(self._ctx, int(step), C.byref(hp), _stream_ptr(stream)))

    def apply_step_sgd(self, step, lr=1e-2, momentum=0.9, weight_decay=0.0, stream=None):
        hp = cm_sgd(lr, momentum, weight_decay)
        self._check(lib().cm_apply_step_sgd(self._ctx, int(step), C.byref(hp), _stream_ptr(stream)))

    def apply_bucket(self, bucket, step, lr=1e-3, beta1=0.9, beta2=0.999, eps=1e-8, weight_decay=0.01, stream=None):
        hp = cm_adamw(lr, beta1, beta2, eps, weight_decay)
        self._check(lib().cm_apply_bucket(self._ctx, int(bucket), int(step), C.byref(hp), _stream_ptr(stream)))

    def apply_bucket_sgd(self, bucket, step, lr=1e-2, momentum=0.9, weight_decay=0.0, stream=None):
        hp = cm_sgd(lr, momentum, weight_decay)
        self._check(lib().cm_apply_bucket_sgd(self._ctx, int(bucket), int(step), C.byref(hp), _stream_ptr(stream)))

    def shadow_apply(self, step, stream=None):
        self._check(lib().cm_shadow_apply(self._ctx, int(step), _stream_ptr(stream)))

    def restore(self, stream=None) -> int:
        out = C.c_int64(-1)
        self._check(lib().cm_restore(self._ctx, C.byref(out), _stream_ptr(stream)))
        return out.value

    def gen_grads(self, seed, iteration, scale, stream=None):
        self._check(lib().cm_gen_grads(self._ctx, int(seed), int(iteration), int(scale), _stream_ptr(stream)))

    def init_state(self, seed, stream=None):
        self._check(lib().cm_init_state(self._ctx, int(seed), _stream_ptr(stream)))

    def verify(self, stream=None) -> int:
        out = C.c_int64(-2)
        st = lib().cm_verify(self._ctx, C.byref(out), _stream_ptr(stream))
        if st not in (CM_OK, CM_ERR_INVARIANT):
            self._check(st)
        return out.value

    def verify_ex(self, scope=CM_VERIFY_ALL, stream=None):
        """cm_verify_ex -> (status, mismatch flat index or -1, what: None/'p'/'m'/'v'/'ring'/
        'nonfinite'/'log_gap').  CM_OK and CM_ERR_INVARIANT are returned, others raise."""
        out = C.c_int64(-2)
        what = C.c_int32(-2)
        st = lib().cm_verify_ex(self._ctx, int(scope), C.byref(out), C.byref(what), _stream_ptr(stream))
        if st not in (CM_OK, CM_ERR_INVARIANT):
            self._check(st)
        return st, out.value, VERIFY_WHAT.get(what.value, what.value)

    def barrier(self, stream=None):
        self._check(lib().cm_barrier(self._ctx, _stream_ptr(stream)))

    def check(self):
        """cm_check -> (status, first flagged step or -1, flat index or -1); no synchronisation."""
        st_, ix = C.c_int64(-1), C.c_int64(-1)
        st = lib().cm_check(self._ctx, C.byref(st_), C.byref(ix))
        if st not in (CM_OK, CM_ERR_INVARIANT):
            self._check(st)
        return st, st_.value, ix.value

    def info(self) -> cm_info:
        i = cm_info()
        self._check(lib().cm_get_info(self._ctx, C.byref(i)))
        return i

    def bucket_info(self, b):
        o, p, u = C.c_int64(), C.c_int64(), C.c_int64()
        self._check(lib().cm_bucket_info(self._ctx, int(b), C.byref(o), C.byref(p), C.byref(u)))
        return o.value, p.value, u.value

    def shadow_view(self, half):
        p, m, v = C.c_void_p(), C.c_void_p(), C.c_void_p()
        self._check(lib().cm_shadow_view(self._ctx, int(half), C.byref(p), C.byref(m), C.byref(v)))
        return p.value, m.value, v.value

    def ring_view(self, slot):
        g = C.c_void_p()
        self._check(lib().cm_ring_view(self._ctx, int(slot), C.byref(g)))
        return g.value

    def join(self, stream=None):
        self._check(lib().cm_join(self._ctx, _stream_ptr(stream)))

    def set_param(self, key, value):
        self._check(lib().cm_set_param(self._ctx, key.encode(), int(value)))

    def timing(self, enable):
        """enable=True starts per-kernel timing; enable=False returns (ms[7], counts[7]):
        classes 0-4 kernels (all-reduce, AdamW, shadow AdamW, gen, restore copy), 5 tap
        drains, 6 snapshot persists."""
        ms = (C.c_double * 7)()
        cnt = (C.c_int64 * 7)()
        self._check(lib().cm_timing(self._ctx, 1 if enable else 0, ms, cnt))
        return list(ms), list(cnt)

    def timing_bytes(self):
        """device->host bytes per cm_timing class in the last closed window."""
        b = (C.c_int64 * 7)()
        self._check(lib().cm_timing_bytes(self._ctx, b))
        return list(b)

    def finalize(self):
        if self._ctx:
            lib().cm_finalize(self._ctx)
            self._ctx = C.c_void_p()

    def __del__(self):
        try:
            self.finalize()
        except Exception:
            pass
