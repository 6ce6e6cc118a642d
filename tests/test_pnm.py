"""PNM input (load_pnm, pnm.cpp:124-153) against the unmodified
reference compiled into oracle/_ref: same image, or same error class, message and
byte offset.  Host-side formats (P1/P2/P4 decoding, every header and truncation
error) run here on the CPU; the device P5 pack and the PNM scan are GPU tests."""
import numpy as np
import pytest

from pnm_cases import broken_files, valid_files


def ours(y, data, threshold=128):
    try:
        img = y.load_pnm(data, threshold)
        return ("ok", img.bytes().reshape(img.height, img.row_stride)[:, :(img.width + 7) // 8], img.width, img.height)
    except y.ParseError as e:
        return ("parse", str(e).split(": ", 1)[1], e.offset)
    except y.ValidationError as e:
        return ("invalid", str(e).split(": ", 1)[1])


def same(a, b):
    if a[0] != b[0]:
        return False
    if a[0] == "ok":
        return a[2:] == b[2:] and np.array_equal(a[1], b[1])
    return a[1:] == b[1:]


def test_pnm_known_answers(y):
    # test_imagekit.cpp:172-215
    img = y.load_pnm(b"P1\n2 2\n1 0\n0 1\n")
    assert (img.get(0, 0), img.get(1, 0), img.get(0, 1), img.get(1, 1)) == (True, False, False, True)
    assert y.load_pnm(b"P1 # binary\n2 2 # dims\n1001") == img
    g = y.load_pnm(b"P2\n3 1\n255\n0 127 128\n")
    assert [g.get(x, 0) for x in range(3)] == [True, True, False]
    assert not any(y.load_pnm(b"P2\n3 1\n255\n0 127 128\n", 0).get(x, 0) for x in range(3))
    p4 = y.load_pnm(b"P4\n3 1\n" + bytes([0xBF]))
    assert p4.bytes().ravel().tolist() == [0xA0]  # padding bits forced to background
    assert y.save_pnm(y.BinaryImage(0, 0)) == b"P4\n0 0\n"
    fr = y.load_pnm(b"P4\n5 5\n" + bytes([0xF8, 0x88, 0x88, 0x88, 0xF8]))
    assert y.load_pnm(y.save_pnm(fr)) == fr
    with pytest.raises(y.ValidationError):
        y.load_pnm(b"P2\n1 1\n255\n0\n", 256)
    with pytest.raises(y.ParseError) as e:
        y.load_pnm(b"P5 2 2 255\n" + bytes([1, 2]))
    assert e.value.offset == 11


def test_pnm_host_formats_match_reference(y, ref):
    rng = np.random.default_rng(77)
    good = valid_files(rng, 240)
    for data in good + broken_files(rng, good):
        for thr in (128, 0, 200):
            want = ref.load_pnm(data, thr)
            if want[0] == "ok" and data[:2] == b"P5":
                continue  # valid P5 decodes on the device: tests/test_gpu_pnm.py
            got = ours(y, data, thr)
            assert same(got, want), (data[:40], got[:2], want[:2])
