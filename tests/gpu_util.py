"""Helpers for the GPU parity tests: read the library's host-side views (ring slots, shadow
halves) into numpy and map between the shard-local and flat layouts."""
import ctypes as C

import numpy as np


def host_array(ptr, count, dtype):
    nbytes = count * np.dtype(dtype).itemsize
    buf = (C.c_uint8 * nbytes).from_address(ptr)
    return np.frombuffer(buf, dtype=dtype, count=count).copy()


def shard_slices(rank_obj):
    """[(flat_lo, flat_hi, shard_lo)] for this rank's shard of every bucket."""
    out = []
    n, r = rank_obj.n, rank_obj.rank
    for b in range(rank_obj.n_buckets):
        off, padded, used = rank_obj.ctx.bucket_info(b)
        e = padded // n
        out.append((off + r * e, off + (r + 1) * e, off // n))
    return out


def assemble(group, per_rank_local):
    """Flat array from every rank's shard-local array."""
    r0 = group.ranks[0]
    total = r0.padded
    out = np.zeros(total, per_rank_local[0].dtype)
    for rk, loc in zip(group.ranks, per_rank_local):
        for lo, hi, s in shard_slices(rk):
            out[lo:hi] = loc[s:s + (hi - lo)]
    return out


def ring_flat(group, slot):
    info = group.ranks[0].ctx.info()
    dt = np.float32 if info.grad_dtype == 0 else np.uint16
    locs = [host_array(r.ctx.ring_view(slot), info.shard_numel, dt) for r in group.ranks]
    return assemble(group, locs)


def shadow_flat(group, half):
    info = group.ranks[0].ctx.info()
    outs = []
    for a in range(3):
        locs = [host_array(r.ctx.shadow_view(half)[a], info.shard_numel, np.float32) for r in group.ranks]
        outs.append(assemble(group, locs))
    return outs


def t2np(t):
    import torch
    if t.dtype == torch.bfloat16:
        return t.view(torch.int16).cpu().numpy().view(np.uint16)
    return t.cpu().numpy()


def bits(a):
    a = np.asarray(a)
    return a.view(np.uint32) if a.dtype == np.float32 else a


def host_view(ptr, count, dtype):
    """Zero-copy numpy view of host memory (a ring slot or a host snapshot half)."""
    nbytes = count * np.dtype(dtype).itemsize
    buf = (C.c_uint8 * nbytes).from_address(ptr)
    return np.frombuffer(buf, dtype=dtype, count=count)


def flat_to_local(rank_obj_list, flat_idx):
    """flat indices -> (owner rank, shard-local index) arrays, from the library's bucket table."""
    r0 = rank_obj_list[0]
    n = r0.n
    offs, pads = [], []
    for b in range(r0.n_buckets):
        off, padded, _ = r0.ctx.bucket_info(b)
        offs.append(off)
        pads.append(padded)
    offs, pads = np.asarray(offs, np.int64), np.asarray(pads, np.int64)
    flat_idx = np.asarray(flat_idx, np.int64)
    b = np.searchsorted(offs, flat_idx, side="right") - 1
    e = pads[b] // n
    within = flat_idx - offs[b]
    owner = within // e
    local = offs[b] // n + within - owner * e
    return owner, local


def local_to_flat(rank_obj, local):
    """shard-local index of rank_obj's shard -> flat index."""
    for lo, hi, s in shard_slices(rank_obj):
        if s <= local < s + (hi - lo):
            return lo + (local - s)
    raise IndexError(local)


def flip_host_bit(ptr, index, dtype=np.uint32, bit=0):
    """Flip one bit of element `index` of a host array in place (zero-copy)."""
    a = host_view(ptr, index + 1, dtype)
    a[index] ^= dtype(1 << bit)
