"""Shadow serving client (SPEC.md:422-430 serve_checkpoint, SPEC.md:411-421
consolidate; sec 4.2.4 "each shadow node serves as a checkpoint to the
training nodes simultaneously").

The n shadow shards live in the host segments of ranks 0..n-1 (shard-local order: shard r of
bucket b at element off_b/n).  A trainer -- of this job, of a restarted job, or an evaluator --
fetches the consolidated checkpoint by asking every shard for its slices in parallel
(cm_shadow_serve, one request per bucket shard, each CRC-32 checked) and placing them in the
model's flat bucket-ordered layout; or it fetches one tensor ("layer range") by asking only
the shards that own a piece of it.

Plumbing only: index arithmetic and copies.  The bytes come from cm_shadow_serve.
"""
from __future__ import annotations

from concurrent.futures import ThreadPoolExecutor

import numpy as np

from . import cm

WHAT = {"p": 0, "m": 1, "v": 2}


class ShardMap:
    """The plan's bucket table and the shard each rank owns (SURVEY 8.e partition)."""

    def __init__(self, numel, grad_dtype, cap_bytes, world_size):
        self.n = int(world_size)
        self.numel = [int(x) for x in numel]
        self.padded, _, self.tensor_off = cm.plan_buckets(self.numel, grad_dtype, cap_bytes, self.n)
        self.buckets = cm.plan_bucket_table(self.numel, grad_dtype, cap_bytes, self.n)   # (off, E_b, used)
        self.shard_numel = sum(E // self.n for _, E, _ in self.buckets)

    def pieces(self, lo, hi):
        """Split the global flat range [lo, hi) into (rank, shard-local off, global off, count)."""
        out = []
        for off, E, _ in self.buckets:
            if hi <= off or lo >= off + E:
                continue
            s = E // self.n
            for r in range(self.n):
                a, b = max(lo, off + r * s), min(hi, off + (r + 1) * s)
                if a < b:
                    out.append((r, off // self.n + (a - off - r * s), a, b - a))
        return out


def consolidate(shm_name, world_size):
    """The step every shard can serve: min over shards of the newest snapshot (cm_shadow_consolidate)."""
    return cm.shadow_consolidate(shm_name, world_size)


def _check_layout(shm_name, smap):
    for r in range(smap.n):
        d = cm.shadow_query(shm_name, r)
        if d.world_size != smap.n or d.shard_numel != smap.shard_numel:
            raise cm.CMError(cm.CM_ERR_CONFIG, f"segment {shm_name}.r{r}: world {d.world_size}, shard "
                             f"{d.shard_numel} elements; the plan says {smap.n} / {smap.shard_numel}")


def _serve_into(shm_name, step, what, pieces, dst, base, verify, threads):
    """Serve every (rank, shard-local off, global off, count) piece into dst[global - base]."""
    def one(piece):
        r, loc, g, cnt = piece
        view = dst[g - base:g - base + cnt]
        _, crc = cm.shadow_serve(shm_name, r, step, what, loc, cnt, out=view)
        if verify and crc != cm.crc32(view):
            raise cm.CMError(cm.CM_ERR_INVARIANT, f"rank {r} [{loc}, {loc + cnt}): CRC-32 mismatch")
        return cnt
    with ThreadPoolExecutor(max_workers=threads) as ex:   # ctypes releases the GIL: shards in parallel
        return sum(ex.map(one, pieces))


def _split(pieces, chunk):
    out = []
    for r, loc, g, cnt in pieces:
        for k in range(0, cnt, chunk):
            c = min(chunk, cnt - k)
            out.append((r, loc + k, g + k, c))
    return out


def fetch(shm_name, smap: ShardMap, step=None, what=("p", "m", "v"), threads=8, verify=True,
          chunk_elems=16 << 20):
    """Fetch the whole checkpoint at `step` (default: the consolidated step) from all shards.
    Returns (step, {name: float32 array of padded_numel elements in the flat layout})."""
    _check_layout(shm_name, smap)
    if step is None:
        step = consolidate(shm_name, smap.n)
    pieces = _split(smap.pieces(0, smap.padded), chunk_elems)
    out = {}
    for w in what:
        dst = np.zeros(smap.padded, dtype=np.float32)
        _serve_into(shm_name, step, WHAT[w], pieces, dst, 0, verify, threads)
        out[w] = dst
    return step, out


def fetch_tensor(shm_name, smap: ShardMap, index, step=None, what="p", verify=True):
    """Fetch one tensor (a "layer range") at `step` from the shards owning it."""
    if step is None:
        step = consolidate(shm_name, smap.n)
    lo = smap.tensor_off[index]
    hi = lo + smap.numel[index]
    dst = np.empty(hi - lo, dtype=np.float32)
    pieces = smap.pieces(lo, hi)
    _serve_into(shm_name, step, WHAT[what], pieces, dst, lo, verify, threads=4)
    return step, dst


def export(shm_name, numel, grad_dtype, cap_bytes, world_size, path, step=None):
    """Write the checkpoint at `step` (default: consolidated) as a per-tensor model file
    (cm_shadow_export); returns the step written."""
    return cm.shadow_export(shm_name, numel, grad_dtype, cap_bytes, world_size, path, -1 if step is None else step)


MODEL_MAGIC = 0x4C444F4D5442434B     # "KCBTMODL"


def read_model_file(path, verify=True):
    """Parse a cm_shadow_export file (layout in include/cm.h) -> (header dict, [records]);
    each record {"index", "p", "m", "v"}.  verify: the file CRC-32 and every array's."""
    import struct
    import zlib
    raw = open(path, "rb").read()
    magic, ver, nt, world, dtype, step, lh, cap, crc = struct.unpack_from("<QIiiiqQqI", raw, 0)
    if magic != MODEL_MAGIC or ver != 1:
        raise ValueError(f"{path}: not a model checkpoint file")
    if verify and zlib.crc32(raw[64:]) != crc:
        raise ValueError(f"{path}: CRC-32 mismatch")
    hdr = {"n_tensors": nt, "world_size": world, "dtype": dtype, "step": step, "layout_hash": lh, "cap_bytes": cap}
    recs, o = [], 64
    for _ in range(nt):
        idx, n, c0, c1, c2 = struct.unpack_from("<qqIII", raw, o)
        o += 32
        arrs = {}
        for w, c in zip("pmv", (c0, c1, c2)):
            a = np.frombuffer(raw, dtype=np.float32, count=n, offset=o)
            if verify and zlib.crc32(a.tobytes()) != c:
                raise ValueError(f"{path}: tensor {idx} {w}: CRC-32 mismatch")
            arrs[w] = a
            o += 4 * n
        recs.append({"index": idx, **arrs})
    if o != len(raw):
        raise ValueError(f"{path}: {len(raw) - o} trailing bytes")
    return hdr, recs
