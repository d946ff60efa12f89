"""FBSIDX1 index files (bench/persist.py; reference tests test_bench.py:80-167).
Golden files in tests/golden/idx were written by the reference's own
save_index (tests/golden/make_golden_persist.py)."""

import struct
import zlib
from pathlib import Path

import numpy as np
import pytest

from oracle import fs_oracle as orc
from paper_1506_08620_b200 import persist
from paper_1506_08620_b200.errors import BadMagic, ChecksumMismatch, TruncatedFile, VersionMismatch

IDX = Path(__file__).resolve().parent / "golden" / "idx"
FILES = sorted(IDX.glob("*.idx"))


def _ref_fields(raw: bytes):
    hd = persist.parse_header(raw)
    k = np.frombuffer(raw, dtype="<u4", count=hd["r"] + 1, offset=48)
    (crc,) = struct.unpack("<I", raw[hd["end"]:hd["end"] + 4])
    return hd, k, crc


# ---------------------------------------------------------------- CPU ----


@pytest.mark.parametrize("path", FILES, ids=[f.stem for f in FILES])
def test_golden_files_parse_and_match_oracle(path):
    raw = path.read_bytes()
    hd, k, crc = _ref_fields(raw)
    assert zlib.crc32(k.tobytes()) == crc
    assert len(raw) == 48 + 4 * (hd["r"] + 1) + 4


def test_header_errors_in_reference_order(tmp_path):
    raw = (IDX / "s100_double.idx").read_bytes()
    with pytest.raises(BadMagic):
        persist.parse_header(b"NOTANIDX" + b"\0" * 64)
    for cut in (4, 20, len(raw) - 3):
        with pytest.raises(TruncatedFile):
            persist.parse_header(raw[:cut])
    bad = bytearray(raw)
    bad[8] = 99
    with pytest.raises(VersionMismatch):
        persist.parse_header(bytes(bad))
    bad = bytearray(raw)
    bad[11] = 16  # qbits
    with pytest.raises(VersionMismatch):
        persist.parse_header(bytes(bad))


# ---------------------------------------------------------------- GPU ----


@pytest.mark.gpu
@pytest.mark.parametrize("path", FILES, ids=[f.stem for f in FILES])
def test_gpu_load_and_save_byte_identical(cuda, path, tmp_path):
    raw = path.read_bytes()
    hd, k, _ = _ref_fields(raw)
    idx = persist.load_index(path)
    assert np.array_equal(idx.k, k) and idx.k.dtype == np.uint32
    assert (idx.r, idx.n, idx.q, idx.qbits, idx.precision) == (hd["r"], hd["n"], hd["q"], hd["qbits"], hd["precision"])
    assert len(idx.left_pad) == idx.q - 1
    out = tmp_path / "back.idx"
    assert persist.save_index(idx, out) == len(raw)
    assert out.read_bytes() == raw


@pytest.mark.gpu
def test_gpu_round_trip_search_identical(cuda, tmp_path):
    import paper_1506_08620_b200 as fs

    p = fs.gen_uniform_gap_partition(100, 1, 5, seed=31, precision="double")
    z = np.concatenate([orc.random_queries(p.values, 20_000, seed=4), orc.boundary_probes(p.values)])
    want = orc.rank_oracle(p.values, z)
    for q, algo in ((1, "direct"), (2, "direct-gap2"), (3, "direct-generic"), (5, "direct-generic")):
        idx, _ = fs.build(p, q=q)
        path = tmp_path / f"t{q}.idx"
        persist.save_index(idx, path)
        back = persist.load_index(path)
        assert back.h == idx.h and back.h.dtype == idx.h.dtype and back.x0 == idx.x0 and back.q == q
        # the kernel follows the file's gap (default), and an explicit name must agree with it
        assert persist.prepare_loaded(back, p).algorithm == algo
        assert np.array_equal(fs.run_batch(persist.prepare_loaded(back, p), z), want), q
        assert np.array_equal(fs.run_batch(persist.prepare_loaded(back, p, algo), z), want), q
        for wrong in {"direct", "direct-gap2", "direct-generic"} - {algo}:
            with pytest.raises(ValueError):
                persist.prepare_loaded(back, p, wrong)


@pytest.mark.gpu
def test_gpu_loaded_index_gets_prepares_layouts(cuda, tmp_path):
    """A loaded gap-1 index is searched through the same shared-memory layouts
    prepare() builds over a fresh table (persist.prepare_loaded calls
    batch.set_direct_layouts): cfg3's fused records, cfg5 N+1 = 1025's count
    words beside X (K: 33 MB on disk) and cfg4's striped rank words, with
    identical placements and the oracle's answers."""
    import paper_1506_08620_b200 as fs
    from paper_1506_08620_b200 import workloads

    for name, kw in (("cfg3", {}), ("cfg5", {"n1": 1025}), ("cfg4", {})):
        p = workloads.knots(name, **kw)
        fresh = fs.prepare("direct", p)
        path = tmp_path / f"{name}.idx"
        persist.save_index(fresh.structure, path)
        loaded = persist.prepare_loaded(persist.load_index(path), p)
        path.unlink()
        assert loaded.placement() == fresh.placement(), name
        assert loaded.placement()["smem_table"] or loaded.placement()["smem_sparse"], name
        z = np.concatenate([workloads.queries_host(name, p, 200_000, seed=3), orc.boundary_probes(p.values)])
        z = z[(z >= p.values[0]) & (z < p.values[-1])].astype(p.values.dtype)
        want = orc.rank_oracle(p.values, z)
        assert np.array_equal(fs.run_batch(loaded, z), want), name
        assert np.array_equal(fs.run_batch(fresh, z), want), name


@pytest.mark.gpu
def test_gpu_corrupt_payload_detected(cuda, tmp_path):
    raw = bytearray((IDX / "s100_double.idx").read_bytes())
    raw[60] ^= 0xFF
    path = tmp_path / "c.idx"
    path.write_bytes(bytes(raw))
    with pytest.raises(ChecksumMismatch):
        persist.load_index(path)


@pytest.mark.gpu
@pytest.mark.parametrize("nbytes", [1, 3, 4, 5, 4095, 4096, 4097, 8192, 12289, 1 << 20, (1 << 20) + 7, 100_000_003])
def test_gpu_crc32_equals_zlib(cuda, nbytes):
    import torch

    rng = np.random.default_rng(nbytes)
    host = rng.integers(0, 256, size=nbytes, dtype=np.uint8)
    t = torch.from_numpy(host).to(cuda)
    assert persist.device_crc32(t) == zlib.crc32(host.tobytes())
    # unaligned start
    if nbytes > 5:
        assert persist.device_crc32(t[3:]) == zlib.crc32(host[3:].tobytes())
