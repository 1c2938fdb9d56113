"""CheckpointFile persistence of the host shadow, on the
CPU: save/load round trip of a shadow segment, CRC-32 equal to zlib's, corruption refused."""
import os
import struct
import zlib

import numpy as np
import pytest

from paper_2507_13522_b200 import cm

SEG_MAGIC = 0x434B4D5442323030


def _fake_segment(name, size, seed=0):
    rng = np.random.default_rng(seed)
    buf = bytearray(rng.integers(0, 256, size, dtype=np.uint8).tobytes())
    struct.pack_into("<Q", buf, 0, SEG_MAGIC)          # SegHeader.magic
    struct.pack_into("<I", buf, 8, 2)                  # SegHeader.version
    struct.pack_into("<ii", buf, 12, 1, 0)             # world_size, rank
    struct.pack_into("<q", buf, 56, 7)                 # shadow_step
    struct.pack_into("<Q", buf, 48, 0x1234)            # layout_hash
    struct.pack_into("<Q", buf, 112, size)             # total
    with open(f"/dev/shm/{name}.r0", "wb") as f:
        f.write(buf)
    return bytes(buf)


def test_crc32_matches_zlib():
    rng = np.random.default_rng(1)
    for n in (0, 1, 7, 8, 9, 4096, 100003):
        data = rng.integers(0, 256, n, dtype=np.uint8).tobytes()
        assert cm.crc32(data) == zlib.crc32(data)


def test_save_load_round_trip_and_corruption(tmp_path):
    name = f"cmfile{os.getpid()}"
    payload = _fake_segment(name, 1 << 20)
    path = tmp_path / "shadow.ckpt"
    try:
        cm.shadow_save(name, 0, path)
        raw = path.read_bytes()
        magic, ver, crc, nbytes = struct.unpack_from("<QIIQ", raw, 0)
        assert ver == 1 and nbytes == len(payload) and raw[64:] == payload
        assert crc == zlib.crc32(payload)
        cm.unlink_shadow(name, 0)
        cm.shadow_load(path, name + "x", 0)
        with open(f"/dev/shm/{name}x.r0", "rb") as f:
            assert f.read() == payload
        cm.unlink_shadow(name + "x", 0)
        bad = bytearray(raw)
        bad[64 + 12345] ^= 0x40                         # flip one payload bit
        path.write_bytes(bytes(bad))
        with pytest.raises(cm.CMError) as e:
            cm.shadow_load(path, name + "y", 0)
        assert e.value.status == cm.CM_ERR_INVARIANT
        assert not os.path.exists(f"/dev/shm/{name}y.r0")
        with pytest.raises(cm.CMError):
            cm.shadow_load(path, name + "z", 1)         # wrong rank
        # a header that claims more payload than the file holds is refused before any
        # segment is created (never size a segment from an untrusted header)
        trunc = bytearray(raw[:-4096])
        path.write_bytes(bytes(trunc))
        with pytest.raises(cm.CMError) as e:
            cm.shadow_load(path, name + "z", 0)
        assert e.value.status == cm.CM_ERR_ARG
        assert not os.path.exists(f"/dev/shm/{name}z.r0")
        # a payload whose segment header describes another segment (total, layout)
        other = bytearray(raw)
        struct.pack_into("<Q", other, 64 + 112, len(payload) + 4096)
        path.write_bytes(bytes(other))
        with pytest.raises(cm.CMError) as e:
            cm.shadow_load(path, name + "z", 0)
        assert e.value.status == cm.CM_ERR_INVARIANT
        assert not os.path.exists(f"/dev/shm/{name}z.r0")
    finally:
        for suffix in ("", "x", "y", "z"):
            try:
                os.unlink(f"/dev/shm/{name}{suffix}.r0")
            except FileNotFoundError:
                pass
