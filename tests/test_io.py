"""CPU: frame / track-log I/O of SURVEY §8(f) row 3 (host side of the
library, no device needed): PNM decoding, frame-sequence ingest and the
track-log text interchange match the reference byte for byte, including the
IoError messages (golden tests/golden/io.npz from the reference; live
comparison with oracle/_ref when present)."""
import ctypes as C
import os

import numpy as np
import pytest

import paper_1310_3322_b200 as trb
from paper_1310_3322_b200.api import IoError
from tests import _oracle as O
from tests.golden.make_golden import PNM_CASES

GOLD = os.path.join(os.path.dirname(__file__), "golden")
needs_ref = pytest.mark.skipif(not O.ref_available(), reason="oracle/_ref not built")


def test_decode_pnm_golden():
    g = np.load(os.path.join(GOLD, "io.npz"))
    off = 0
    for b, (w, h, c), err in zip(PNM_CASES, g["pnm_dims"], g["pnm_errors"]):
        if err:
            with pytest.raises(IoError) as e:
                trb.decode_pnm(b)
            assert str(e.value) == err
        else:
            px, w2, h2, c2 = trb.decode_pnm(b)
            n = w * h * c
            assert (w2, h2, c2) == (w, h, c)
            assert px.tobytes() == g["pnm_pixels"][off:off + n].tobytes()
            off += n


def test_track_log_text_golden(tmp_path):
    g = np.load(os.path.join(GOLD, "io.npz"))
    log = g["log"]
    text = trb.format_track_log(log)
    assert text.encode() == bytes(g["log_text"])
    back = trb.parse_track_log(text)
    assert back.tobytes() == log.tobytes()
    p = tmp_path / "tracks.txt"
    trb.save_track_log(log, str(p))
    assert p.read_bytes() == bytes(g["log_text"])
    assert trb.load_track_log(str(p)).tobytes() == log.tobytes()


def test_track_log_parse_errors():
    ok = "# c\n\n  \t\n0 1 2.5 3 4 5 lost\n"
    a = trb.parse_track_log(ok)
    assert len(a) == 1 and a["status"][0] == trb.LOST and a["x"][0] == 2.5
    with pytest.raises(IoError, match=r"bad track log record at <memory>:2"):
        trb.parse_track_log("# h\n0 1 2 3 4\n")
    with pytest.raises(IoError, match=r"unknown track status 'gone' at src:1"):
        trb.parse_track_log("0 1 2 3 4 5 gone\n", "src")
    with pytest.raises(IoError, match="cannot open"):
        trb.load_track_log("/nonexistent/dir/x.txt")


def _write_sequence(d, names, w=3, h=2, c=1, seed=0):
    rng = np.random.default_rng(seed)
    frames = {}
    for nm in names:
        px = rng.integers(0, 256, size=w * h * c, dtype=np.uint8)
        magic = b"P5" if c == 1 else b"P6"
        (d / nm).write_bytes(magic + f"\n{w} {h}\n255\n".encode() + px.tobytes())
        frames[nm] = px
    return frames


def test_load_frame_sequence(tmp_path):
    names = ["frame_000010.pgm", "frame_000002.pgm", "frame_000007.pgm", "cam.pgm", "notes.txt"]
    (tmp_path / "notes.txt").write_text("ignored")
    fr = _write_sequence(tmp_path, names[:4])
    out, idx, w, h, c = trb.load_frame_sequence(str(tmp_path))
    # stems without trailing digits take their position in path order
    # ("cam.pgm" sorts first -> index 0); then ordered by index
    assert (w, h, c) == (3, 2, 1)
    assert idx.tolist() == [0, 2, 7, 10]
    assert [out[i].tobytes() for i in range(4)] == [fr[n].tobytes() for n in
                                                    ["cam.pgm", "frame_000002.pgm", "frame_000007.pgm",
                                                     "frame_000010.pgm"]]
    _write_sequence(tmp_path, ["frame_000011.ppm"], c=3)
    with pytest.raises(IoError, match=r"dimension mismatch in .*frame_000011.ppm: expected 3x2x1, got 3x2x3"):
        trb.load_frame_sequence(str(tmp_path))
    with pytest.raises(IoError, match="not a directory"):
        trb.load_frame_sequence(str(tmp_path / "nope"))


@needs_ref
def test_io_vs_reference(tmp_path):
    L = O.ref_lib()
    for b in PNM_CASES + [b"P6\n1 1\n255\n\x01\x02\x03", b"P5 2 1 255\n\x00"]:
        buf = np.frombuffer(b, np.uint8) if b else np.zeros(1, np.uint8)
        w, h, c = C.c_int(0), C.c_int(0), C.c_int(0)
        out = np.zeros(64, np.uint8)
        rc = L.ref_decode_pnm(buf.ctypes.data, len(b), b"<memory>", C.byref(w), C.byref(h), C.byref(c),
                              out.ctypes.data, out.size)
        if rc:
            with pytest.raises(IoError) as e:
                trb.decode_pnm(b)
            assert str(e.value) == L.ref_last_error().decode()
        else:
            px, *dims = trb.decode_pnm(b)
            assert dims == [w.value, h.value, c.value]
            assert px.tobytes() == out[:px.size].tobytes()
    names = ["b_3.pgm", "a_3.pgm", "z.pgm", "y.pgm", "x_01.pgm", "x_1.pgm", "q9.pgm"]
    _write_sequence(tmp_path, names, seed=4)
    n, w, h, c = C.c_int(0), C.c_int(0), C.c_int(0), C.c_int(0)
    idx = np.zeros(16, np.int64)
    ref = np.zeros(16 * 6, np.uint8)
    assert L.ref_load_frame_sequence(str(tmp_path).encode(), C.byref(n), C.byref(w), C.byref(h), C.byref(c),
                                     idx.ctypes.data, ref.ctypes.data, ref.size) == 0
    out, ours_idx, *_ = trb.load_frame_sequence(str(tmp_path))
    assert ours_idx.tolist() == idx[:n.value].tolist()
    assert out.tobytes() == ref[:out.size].tobytes()
    text = "0 1 0.1 0.2 3 4 active\n5 6 1e-310 -2.5e300 7 8 lost\n"
    res = np.zeros(4, trb.api.LOG_DTYPE)
    nn = C.c_int64(0)
    assert L.ref_parse_track_log(text.encode(), len(text), b"s", res.ctypes.data, 4, C.byref(nn)) == 0
    assert trb.parse_track_log(text, "s").tobytes() == res[:nn.value].tobytes()
