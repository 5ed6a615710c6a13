"""f-2 image ingestion (image.cpp:40-138): the native loader against the
reference's own behaviour. Cases restate the reference's test_image.cpp
vectors (byte strings written to disk) and cross-check every accepted and
rejected file against dic::load_image / dic::load_sequence built from the
reference sources (oracle/_ref). No GPU needed."""
import ctypes as C
import os

import numpy as np
import pytest

from paper_1905_06228_b200 import _abi, dic
from paper_1905_06228_b200.dic import DicError

import oracle.pyoracle as po


def _write(path, data: bytes):
    with open(path, "wb") as f:
        f.write(data)
    return path


def _ref_load(path):
    """dic::load_image from the reference build: (pixels, None) or (None, message)."""
    L = C.CDLL(po.PATHS["reference"])
    w, h = C.c_int(), C.c_int()
    err = C.create_string_buffer(512)
    if L.dicref_load_image(str(path).encode(), None, C.c_size_t(0), C.byref(w), C.byref(h), err, 512):
        return None, err.value.decode()
    out = np.zeros(w.value * h.value, np.float64)
    L.dicref_load_image(str(path).encode(), out.ctypes.data_as(C.c_void_p), C.c_size_t(out.size), C.byref(w),
                        C.byref(h), err, 512)
    return out.reshape(h.value, w.value), None


def _ours(path, allow_16bit=False):
    try:
        return dic.load_image(path, allow_16bit).pixels(), None
    except DicError as e:
        return None, str(e)


needs_ref = pytest.mark.skipif(not po.available("reference"), reason="reference build absent")

# test_image.cpp vectors
VECTORS = {
    "p5_identity": b"P5\n2 2\n255\n" + bytes([0x00, 0xFF, 0x80, 0x40]),
    "p5_single": b"P5\n1 1\n255\n\x07",
    "p5_trunc": b"P5\n4 4\n255\n" + b"xxx",
    "p5_zero": b"P5\n0 3\n255\n",
    "p5_deep": b"P5\n2 2\n65535\n....",
    "png": b"\x89PNG....",
    "p2_comment": b"P2\n# comment line\n3 1\n255\n10 20 30\n",
    "p2_range": b"P2\n2 1\n100\n10 101\n",
    "p2_trunc": b"P2\n3 1\n255\n1 2\n",
    "p5_maxval_low": b"P5\n2 1\n15\n\x03\x0f",
    "p5_comment_hdr": b"P5\n# a\n# b\n3 # w\n1\n255\n\x01\x02\x03",
}


def test_reference_vectors_known_answers(tmp_path):
    px, err = _ours(_write(tmp_path / "a.pgm", VECTORS["p5_identity"]))
    assert err is None and px.tolist() == [[0, 255], [128, 64]]
    px, _ = _ours(_write(tmp_path / "b.pgm", VECTORS["p5_single"]))
    assert px.tolist() == [[7]]
    px, _ = _ours(_write(tmp_path / "c.pgm", VECTORS["p2_comment"]))
    assert px.tolist() == [[10, 20, 30]]
    for name, key in (("trunc", "unreadable"), ("zero", "zero-dimension"), ("deep", "unsupported")):
        _, err = _ours(_write(tmp_path / f"{name}.pgm", VECTORS[f"p5_{name}"]))
        assert key in err
    _, err = _ours(_write(tmp_path / "png.pgm", VECTORS["png"]))
    assert err is not None
    _, err = _ours(tmp_path / "missing.pgm")
    assert "unreadable" in err


@needs_ref
@pytest.mark.parametrize("name", sorted(VECTORS))
def test_loader_matches_reference_build(tmp_path, name):
    path = _write(tmp_path / f"{name}.pgm", VECTORS[name])
    got, gerr = _ours(path)
    exp, eerr = _ref_load(path)
    assert (gerr is None) == (eerr is None), (gerr, eerr)
    if eerr is None:
        assert np.array_equal(got.astype(np.float64), exp)
    else:
        assert gerr.split(":")[0] == eerr.split(":")[0]


@needs_ref
def test_random_graymaps_match_reference_build(tmp_path):
    rng = np.random.default_rng(7)
    for i in range(12):
        w, h = int(rng.integers(1, 60)), int(rng.integers(1, 40))
        maxval = int(rng.integers(1, 256))
        px = rng.integers(0, maxval + 1, size=(h, w), dtype=np.int64)
        if i % 2:
            data = f"P5\n{w} {h}\n{maxval}\n".encode() + px.astype(np.uint8).tobytes()
        else:
            data = (f"P2\n# random\n{w} {h}\n{maxval}\n" + " ".join(map(str, px.ravel())) + "\n").encode()
        path = _write(tmp_path / f"r{i}.pgm", data)
        got, _ = _ours(path)
        exp, _ = _ref_load(path)
        assert np.array_equal(got.astype(np.float64), exp) and np.array_equal(got, px)


def test_sixteen_bit_extension(tmp_path):
    """maxval > 255: rejected by default (reference behaviour), read exactly
    (big-endian P5 / ASCII P2) with allow_16bit."""
    rng = np.random.default_rng(3)
    px = rng.integers(0, 4096, size=(5, 7)).astype(np.uint16)
    p5 = _write(tmp_path / "w.pgm", b"P5\n7 5\n4095\n" + px.astype(">u2").tobytes())
    p2 = _write(tmp_path / "w2.pgm", ("P2\n7 5\n4095\n" + " ".join(map(str, px.ravel()))).encode())
    for p in (p5, p2):
        _, err = _ours(p)
        assert "unsupported" in err
        got, err = _ours(p, allow_16bit=True)
        assert err is None and got.dtype == np.uint16 and np.array_equal(got, px)
    bad = _write(tmp_path / "w3.pgm", b"P5\n1 1\n1000\n" + np.array([1001], ">u2").tobytes())
    _, err = _ours(bad, allow_16bit=True)
    assert "out of range" in err


def test_save_round_trip_quantizes(tmp_path):
    px = np.array([[0, 7, 255], [300, 1000, 12]], np.uint16)
    dic.save_pgm(dic.GrayImage(px), tmp_path / "s.pgm")
    back = dic.load_image(tmp_path / "s.pgm").pixels()
    assert back.tolist() == [[0, 7, 255], [255, 255, 12]]


@needs_ref
def test_sequence_order_ids_and_errors(tmp_path):
    for name in ("frame_b.pgm", "frame_a.pgm", "frame_c.pgm", "notes.txt"):
        dic.save_pgm(dic.GrayImage(np.full((2, 3), ord(name[6]), np.uint8)), tmp_path / name)
    os.mkdir(tmp_path / "sub.pgm")  # directories never match
    seq = dic.load_sequence(tmp_path, "*.pgm")
    assert [im.pixels()[0, 0] for im in seq] == [ord("a"), ord("b"), ord("c")]
    assert [im.id() for im in seq] == [0, 1, 2]
    # the reference build agrees on order, ids and pixels
    L = C.CDLL(po.PATHS["reference"])
    n, w, h = C.c_int(), C.c_int(), C.c_int()
    out = np.zeros(3 * 6, np.float64)
    ids = (C.c_int * 8)()
    err = C.create_string_buffer(256)
    assert L.dicref_load_sequence(str(tmp_path).encode(), b"*.pgm", out.ctypes.data_as(C.c_void_p), C.c_size_t(18),
                                  C.byref(n), C.byref(w), C.byref(h), ids, C.c_size_t(8), err, 256) == 0
    assert n.value == 3 and list(ids)[:3] == [0, 1, 2]
    assert np.array_equal(out.reshape(3, 2, 3), np.stack([im.pixels() for im in seq]).astype(np.float64))
    # errors
    only = tmp_path / "only"
    os.mkdir(only)
    dic.save_pgm(dic.GrayImage(np.ones((2, 3), np.uint8)), only / "only.pgm")
    with pytest.raises(DicError, match="insufficient images"):
        dic.load_sequence(only, "*.pgm")
    dic.save_pgm(dic.GrayImage(np.ones((2, 2), np.uint8)), only / "other.pgm")
    with pytest.raises(DicError, match="dimension mismatch"):
        dic.load_sequence(only, "*.pgm")
    with pytest.raises(DicError, match="not a directory"):
        dic.load_sequence(tmp_path / "nope", "*.pgm")


def test_loaded_frames_feed_the_abi(tmp_path):
    """Loaded frames are plain u8/u16 host images of the C-ABI (no GPU call)."""
    px = (np.arange(12, dtype=np.uint8) * 9).reshape(3, 4)
    dic.save_pgm(dic.GrayImage(px), tmp_path / "f.pgm")
    im = dic.load_image(tmp_path / "f.pgm", id=5).as_c()
    assert (im.width, im.height, im.dtype, im.id) == (4, 3, _abi.U8, 5)


@pytest.mark.gpu
def test_loaded_sequence_analyzes_like_in_memory_frames(gpu, tmp_path):
    """Frames written as 16-bit P5 files, read back (pageable and pinned), give
    exactly the displacement fields of the in-memory frames."""
    import copy

    from paper_1905_06228_b200 import configs

    w = configs.crop(configs.c5(5), 160, 144)
    frames = [f.render() for f in w.frames]
    maxv = int(max(f.max() for f in frames))
    for i, f in enumerate(frames):
        _write(tmp_path / f"img_{i:03d}.pgm", f"P5\n{f.shape[1]} {f.shape[0]}\n{maxv}\n".encode() +
               f.astype(">u2").tobytes())
    cfg = copy.deepcopy(w.cfg)
    exp = dic.analyze_sequence([dic.GrayImage(f, i) for i, f in enumerate(frames)], cfg)
    for pinned in (False, True):
        seq = dic.load_sequence(tmp_path, "img_*.pgm", allow_16bit=True, pinned=pinned)
        assert all(np.array_equal(s.pixels(), f) for s, f in zip(seq, frames))
        got = dic.analyze_sequence(seq, cfg)
        for g, e in zip(got, exp):
            assert not g.failed() and (g.ref_id, g.tgt_id) == (e.ref_id, e.tgt_id)
            for k in e.records.dtype.names:
                assert np.array_equal(g.records[k], e.records[k], equal_nan=True), (pinned, k)
