"""Shadow serving on the CPU (SPEC.md:422-430 serve_checkpoint, SPEC.md:411-421
consolidate): host segments of n ranks are written here byte by byte in the library's
segment layout (SegHeader + snapshot halves), each half holding a known global model at a
known step, split into shards by the plan's bucket table (rank r owns [off_b + r E_b/n,
off_b + (r+1) E_b/n) of every bucket, concatenated in bucket order).  Checked:
- the consolidated step is the min rule's, and a shard that advanced past it twice is a
  consolidation failure;
- the full owned range of a shard is exactly the half's bytes, with zlib's CRC-32;
- every shard fetched in parallel reassembles the global model bit-exactly (and one tensor
  from the shards that own it), from several processes at once;
- out-of-range requests and missing steps are refused;
- a half rewritten while it is served is never returned torn (seqlock on its step word)."""
import mmap
import multiprocessing as mp
import os
import struct
import threading
import time
import zlib

import numpy as np
import pytest

from paper_2507_13522_b200 import cm, serving

SEG_MAGIC = 0x434B4D5442323030
NUMEL = [5000, 130000, 7, 64, 90001, 3000]
CAP = 256 << 10


def _global(step, what, padded):
    """The model a half at `step` holds (any finite values; distinct per step / array)."""
    rng = np.random.default_rng(1000 * step + what)
    return rng.standard_normal(padded).astype(np.float32)


def _shard(glob, buckets, n, r):
    return np.concatenate([glob[off + r * (E // n): off + (r + 1) * (E // n)] for off, E, _ in buckets])


def _layout_hash(numel, cap, dtype, n):
    """FNV-1a 64 over the int64 tensor sizes, the int64 cap, the int32 dtype and int32 n
    (the segment header's layout hash, include/cm.h cm_register_buckets)."""
    h = 0xCBF29CE484222325
    for b in np.asarray(numel, np.int64).tobytes() + struct.pack("<qii", cap, dtype, n):
        h = ((h ^ b) * 0x100000001B3) & 0xFFFFFFFFFFFFFFFF
    return h


def _write_segment(name, n, r, halves, layout_hash=None, world=None):
    """halves: [(step, [p, m, v] shard arrays) or (-1, None)] x 2."""
    L = len(next(h[1][0] for h in halves if h[1] is not None))
    if layout_hash is None:
        layout_hash = _layout_hash(NUMEL, CAP, cm.CM_F32, world or n)
    state_off = 4096
    total = (state_off + 6 * L * 4 + 4095) // 4096 * 4096
    buf = bytearray(total)
    struct.pack_into("<QIiiiiiii", buf, 0, SEG_MAGIC, 2, world or n, r, 0, 4, 1, cm.CM_SHADOW_HOST, 0)
    struct.pack_into("<qQq", buf, 40, L, layout_hash, max(h[0] for h in halves))
    struct.pack_into("<qq", buf, 64, halves[0][0], halves[1][0])
    struct.pack_into("<QQQQQ", buf, 80, 4096, 4096, 4096, state_off, total)
    struct.pack_into("<qq", buf, 120, -1, -1)
    for hf, (_, arrs) in enumerate(halves):
        if arrs is None:
            continue
        for a, x in enumerate(arrs):
            o = state_off + (hf * 3 + a) * L * 4
            buf[o:o + L * 4] = x.tobytes()
    with open(f"/dev/shm/{name}.r{r}", "wb") as f:
        f.write(buf)
    return state_off, L


@pytest.fixture
def segs():
    name = f"cmserve{os.getpid()}"
    made = []

    def make(n, steps_per_rank, **kw):
        smap = serving.ShardMap(NUMEL, cm.CM_F32, CAP, n)
        for r in range(n):
            halves = []
            for s in steps_per_rank[r]:
                if s < 0:
                    halves.append((-1, None))
                else:
                    halves.append((s, [_shard(_global(s, a, smap.padded), smap.buckets, n, r) for a in range(3)]))
            _write_segment(name, n, r, halves, **kw)
            made.append(r)
        return name, smap

    yield make
    for r in set(made):
        cm.unlink_shadow(name, r)


def test_consolidate_min_rule(segs):
    name, _ = segs(3, [(16, 8), (8, 0), (16, 24)])
    with pytest.raises(cm.CMError) as e:               # rank 2 advanced past 8 twice
        serving.consolidate(name, 3)
    assert e.value.status == cm.CM_ERR_STATE
    name, _ = segs(3, [(16, 8), (8, 0), (16, 8)])
    assert serving.consolidate(name, 3) == 8
    name, _ = segs(3, [(16, 8), (16, 24), (16, 8)])
    assert serving.consolidate(name, 3) == 16
    name, _ = segs(2, [(0, -1), (8, 0)])
    assert serving.consolidate(name, 2) == 0


def test_consolidate_layout_mismatch(segs):
    name, smap = segs(2, [(4, 2), (4, 2)])
    _write_segment(name, 2, 1, [(4, [np.zeros(smap.shard_numel, np.float32)] * 3), (2, [np.zeros(smap.shard_numel,
                                                                                                  np.float32)] * 3)],
                   layout_hash=0x1)
    with pytest.raises(cm.CMError) as e:
        serving.consolidate(name, 2)
    assert e.value.status == cm.CM_ERR_CONFIG


def test_full_range_is_the_half_and_crc_is_zlib(segs):
    n = 2
    name, smap = segs(n, [(6, 4), (4, 6)])
    for r in range(n):
        for what in range(3):
            want = _shard(_global(4, what, smap.padded), smap.buckets, n, r)
            got, crc = cm.shadow_serve(name, r, 4, what, 0, smap.shard_numel)
            assert got.tobytes() == want.tobytes()
            assert crc == zlib.crc32(want.tobytes())
            part, crc = cm.shadow_serve(name, r, 6, what, 123, 4567)
            want6 = _shard(_global(6, what, smap.padded), smap.buckets, n, r)[123:123 + 4567]
            assert part.tobytes() == want6.tobytes() and crc == zlib.crc32(want6.tobytes())
    _, crc = cm.shadow_serve(name, 0, 4, 0, smap.shard_numel, 0)   # empty request at the end
    assert crc == 0
    d = cm.shadow_query(name, 1)
    assert (d.world_size, d.rank, d.shard_numel, list(d.half_step)) == (2, 1, smap.shard_numel, [4, 6])


def test_device_placed_shadow_is_not_served(segs):
    """A DEVICE-placed shadow has no host snapshot halves: nothing to serve (CM_ERR_ARG)."""
    name, smap = segs(1, [(2, 0)])
    with open(f"/dev/shm/{name}.r0", "r+b") as f:
        f.seek(32)
        f.write(struct.pack("<i", cm.CM_SHADOW_DEVICE))   # SegHeader.shadow_place
    for call in (lambda: cm.shadow_query(name, 0), lambda: cm.shadow_serve(name, 0, 2, 0, 0, 4),
                 lambda: serving.consolidate(name, 1)):
        with pytest.raises(cm.CMError) as e:
            call()
        assert e.value.status == cm.CM_ERR_ARG


def test_requests_refused(segs):
    name, smap = segs(2, [(6, 4), (6, 4)])
    L = smap.shard_numel
    for args, status in [((0, 4, 0, L, 1), cm.CM_ERR_ARG),        # one past the shard
                         ((0, 4, 0, -1, 4), cm.CM_ERR_ARG),
                         ((0, 4, 3, 0, 4), cm.CM_ERR_ARG),        # no such array
                         ((0, 5, 0, 0, 4), cm.CM_ERR_STATE),      # no half holds step 5
                         ((2, 4, 0, 0, 4), cm.CM_ERR_ARG)]:       # no such rank / segment
        r, step, what, off, cnt = args
        with pytest.raises(cm.CMError) as e:
            cm.shadow_serve(name, r, step, what, off, cnt, out=np.empty(max(cnt, 1), np.float32))
        assert e.value.status == status, args
    with pytest.raises(cm.CMError):
        cm.shadow_query(name + "nope", 0)


@pytest.mark.parametrize("n", [1, 2, 4])
def test_fetch_reassembles_the_model(segs, n):
    name, smap = segs(n, [(12, 8)] * (n - 1) + [(8, 4)])
    step, got = serving.fetch(name, smap, threads=n + 1, chunk_elems=50000)
    assert step == 8
    for w, a in serving.WHAT.items():
        np.testing.assert_array_equal(got[w].view(np.uint32), _global(8, a, smap.padded).view(np.uint32))
    for i in range(len(NUMEL)):                         # one tensor at a time ("layer range")
        st, t = serving.fetch_tensor(name, smap, i, what="m")
        lo = smap.tensor_off[i]
        np.testing.assert_array_equal(t.view(np.uint32), _global(8, 1, smap.padded)[lo:lo + NUMEL[i]].view(np.uint32))


@pytest.mark.parametrize("n", [1, 2, 4])
def test_export_model_file(segs, tmp_path, n):
    """the per-tensor model file of the consolidated step holds every
    tensor's p, m, v exactly, each record and the file CRC-32-checked."""
    name, smap = segs(n, [(12, 8)] * (n - 1) + [(8, 4)])
    path = tmp_path / "model.ckpt"
    assert serving.export(name, NUMEL, cm.CM_F32, CAP, n, path) == 8
    hdr, recs = serving.read_model_file(path)
    assert (hdr["step"], hdr["world_size"], hdr["n_tensors"]) == (8, n, len(NUMEL))
    for i, rec in enumerate(recs):
        lo = smap.tensor_off[i]
        assert rec["index"] == i
        for w, a in serving.WHAT.items():
            np.testing.assert_array_equal(rec[w].view(np.uint32),
                                          _global(8, a, smap.padded)[lo:lo + NUMEL[i]].view(np.uint32))
    if n > 1:                                           # the retained half of the leading shards
        with pytest.raises(cm.CMError) as e:
            serving.export(name, NUMEL, cm.CM_F32, CAP, n, path, step=12)
        assert e.value.status == cm.CM_ERR_STATE
    with pytest.raises(cm.CMError) as e:                # another model's table
        serving.export(name, NUMEL[:-1], cm.CM_F32, CAP, n, tmp_path / "x.ckpt")
    assert e.value.status == cm.CM_ERR_CONFIG
    assert not (tmp_path / "x.ckpt").exists() and not (tmp_path / "x.ckpt.tmp").exists()
    raw = bytearray(path.read_bytes())
    raw[64 + 32 + 5] ^= 1                               # one bit of tensor 0's p
    path.write_bytes(bytes(raw))
    with pytest.raises(ValueError):
        serving.read_model_file(path)


def _fetch_worker(name, n, q):
    smap = serving.ShardMap(NUMEL, cm.CM_F32, CAP, n)
    step, got = serving.fetch(name, smap, what=("p", "v"))
    q.put((step, zlib.crc32(got["p"].tobytes()), zlib.crc32(got["v"].tobytes())))


def test_fetch_from_several_trainers_at_once(segs):
    """k shards fetched in parallel by n trainers -> each reassembles the
    consolidated checkpoint."""
    n = 2
    name, smap = segs(n, [(10, 12), (12, 10)])
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    procs = [ctx.Process(target=_fetch_worker, args=(name, n, q)) for _ in range(3)]
    for p in procs:
        p.start()
    outs = [q.get(timeout=120) for _ in procs]
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    want = (12, zlib.crc32(_global(12, 0, smap.padded).tobytes()), zlib.crc32(_global(12, 2, smap.padded).tobytes()))
    assert outs == [want] * 3


def test_never_torn_while_rewritten():
    """A writer rewrites one half over and over the way the shadow does (step word -1, new
    bytes, new step); every served copy either comes back with one step's bytes throughout,
    or is refused with CM_ERR_STATE."""
    name = f"cmtorn{os.getpid()}"
    L = 1 << 21
    state_off, _ = _write_segment(name, 1, 0, [(1, [np.full(L, 1.0, np.float32)] * 3), (-1, None)])
    try:
        with open(f"/dev/shm/{name}.r0", "r+b") as f:
            mm = mmap.mmap(f.fileno(), 0)
        hs = np.frombuffer(mm, dtype=np.int64, count=2, offset=64)
        p = np.frombuffer(mm, dtype=np.float32, count=L, offset=state_off)
        stop = threading.Event()

        def writer():
            s = 1
            while not stop.is_set():
                hs[0] = -1
                s += 1
                p[:L // 2] = s                          # two halves of the copy, a gap between
                p[L // 2:] = s
                hs[0] = s
                time.sleep(0.002)                       # (some copies fit in between)

        th = threading.Thread(target=writer)
        th.start()
        ok = refused = 0
        try:
            out = np.empty(L, np.float32)
            t_end = time.monotonic() + 30.0              # until both outcomes were seen (or 30 s)
            while time.monotonic() < t_end and (ok < 20 or refused < 5):
                s = int(cm.shadow_query(name, 0).half_step[0])
                try:
                    cm.shadow_serve(name, 0, s, 0, 0, L, out=out)
                except cm.CMError as e:
                    assert e.status == cm.CM_ERR_STATE
                    refused += 1
                    continue
                assert out[0] == s and out[-1] == s and (out == s).all(), (s, out[0], out[-1])
                ok += 1
        finally:
            stop.set()
            th.join()
        assert ok > 0 and refused > 0, (ok, refused)
        del hs, p
        mm.close()
    finally:
        cm.unlink_shadow(name, 0)


def test_shard_map_pieces_cover_each_element_once():
    """Property check of the client's range mapping (R31): for random tables, world sizes and
    flat ranges, the pieces tile [lo, hi) exactly once, each inside one rank's shard of one
    bucket, at the shard-local offset the concatenation of that rank's bucket shards gives."""
    from hypothesis import given, settings, strategies as st

    @settings(max_examples=60, deadline=None)
    @given(st.lists(st.integers(1, 5000), min_size=1, max_size=12), st.sampled_from([1, 2, 3, 4, 8]),
           st.sampled_from([cm.CM_F32, cm.CM_BF16]), st.integers(1 << 10, 1 << 14), st.data())
    def prop(numel, n, dtype, cap, data):
        smap = serving.ShardMap(numel, dtype, cap, n)
        lo = data.draw(st.integers(0, smap.padded - 1))
        hi = data.draw(st.integers(lo + 1, smap.padded))
        # reference: global index -> (rank, shard-local index) by concatenating bucket shards
        owner = np.empty(smap.padded, np.int64)
        local = np.empty(smap.padded, np.int64)
        fill = [0] * n
        for off, E, _ in smap.buckets:
            s = E // n
            for r in range(n):
                owner[off + r * s: off + (r + 1) * s] = r
                local[off + r * s: off + (r + 1) * s] = np.arange(fill[r], fill[r] + s)
                fill[r] += s
        assert fill == [smap.shard_numel] * n
        seen = np.zeros(smap.padded, np.int64)
        for r, loc, g, cnt in smap.pieces(lo, hi):
            assert cnt > 0 and lo <= g and g + cnt <= hi
            assert (owner[g:g + cnt] == r).all()
            np.testing.assert_array_equal(local[g:g + cnt], np.arange(loc, loc + cnt))
            seen[g:g + cnt] += 1
        assert (seen[lo:hi] == 1).all() and seen[:lo].sum() == 0 and seen[hi:].sum() == 0

    prop()
