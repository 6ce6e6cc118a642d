"""GPU side of the PNM input path: P5 rasters thresholded and
packed on the device, PNM bytes scanned without a host decode (P4 raster goes to
the device untouched), and the device-resident loader -- against the reference's
load_pnm (oracle/_ref) and the oracle."""
import ctypes

import numpy as np
import pytest

from oracle import Spec
from pnm_cases import valid_files
from test_pnm import ours, same

pytestmark = pytest.mark.gpu


def test_p5_device_decode_matches_reference(gpu, ref):
    y = gpu
    rng = np.random.default_rng(5)
    for data in [f for f in valid_files(rng, 400) if f[:2] == b"P5"]:
        for thr in (0, 1, 128, 255):
            assert same(ours(y, data, thr), ref.load_pnm(data, thr)), data[:30]


def grey_file(bits: np.ndarray, w: int, h: int, rng) -> bytes:
    """A P5 file whose threshold-128 decode is `bits` (dark = foreground)."""
    px = np.unpackbits(bits, axis=1)[:, :w].astype(bool)
    grey = np.where(px, rng.integers(0, 128, size=px.shape), rng.integers(128, 256, size=px.shape)).astype(np.uint8)
    return f"P5\n{w} {h}\n255\n".encode() + grey.tobytes()


@pytest.mark.parametrize("sp", [Spec.random(4099, 3001, 0.5, 3), Spec.hbands(2000, 2000, 147), Spec.checker(777, 555, 7),
                                Spec.frame(1, 1), Spec.random(33, 1, 0.5, 2)])
def test_scan_pnm_all_formats(gpu, orc, sp):
    y = gpu
    rng = np.random.default_rng(sp.width)
    bits = orc.synth(sp)
    want_counts = orc.counts(bits, sp.width)
    he = orc.hyperedges(bits, sp.width)[0]
    img = y.BinaryImage(sp.width, sp.height, bits)
    files = [y.save_pnm(img), grey_file(bits, sp.width, sp.height, rng)]
    if sp.width * sp.height < 200_000:
        px = np.unpackbits(bits, axis=1)[:, :sp.width]
        files.append(f"P1\n{sp.width} {sp.height}\n".encode() + b"\n".join(b" ".join(b"%d" % v for v in r) for r in px))
    for data in files:
        r = y.scan_pnm(data)
        assert np.array_equal(r.counts, want_counts) and r.hyperedges == he, data[:2]
        assert y.load_pnm(data) == img
    # P4 with garbage padding bits: scanned as the reference decodes it (pad = background)
    if sp.width % 8:
        raw = bytearray(files[0])
        hdr = len(raw) - bits.size
        for yy in range(sp.height):
            raw[hdr + yy * bits.shape[1] + bits.shape[1] - 1] |= 0xFF >> (sp.width % 8)
        assert np.array_equal(y.scan_pnm(bytes(raw)).counts, want_counts)


def test_load_pnm_device(gpu, orc):
    y = gpu
    rng = np.random.default_rng(9)
    sp = Spec.random(1001, 257, 0.4, 12)
    bits = orc.synth(sp)
    img = y.BinaryImage(sp.width, sp.height, bits)
    pitch = y.pitch_for(sp.width)
    for data in (y.save_pnm(img), grey_file(bits, sp.width, sp.height, rng)):
        buf = y.DeviceBuffer(pitch * sp.height)
        d = np.frombuffer(data, dtype=np.uint8)
        y._check(y._lib.ychg_load_pnm_device(d.ctypes.data_as(ctypes.c_void_p), d.size, 128, buf.ptr, pitch, None),
                 "load_pnm_device")
        out = buf.to_host(np.zeros((sp.height, pitch), dtype=np.uint8))
        assert np.array_equal(out[:, : bits.shape[1]], bits)
        buf.close()
