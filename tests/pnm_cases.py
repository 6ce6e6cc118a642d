"""PNM byte-string corpus for the loader parity tests (valid files in every
format with comment/whitespace variants, plus truncations and corruptions)."""
import numpy as np


def valid_files(rng: np.random.Generator, count: int) -> list[bytes]:
    out = []
    for i in range(count):
        kind = "1245"[i % 4]
        w, h = int(rng.integers(0, 40)), int(rng.integers(0, 20))
        sep = [b" ", b"\n", b"\t", b"  \n", b" # c\n", b"\r\n"][int(rng.integers(0, 6))]
        head = b"P" + kind.encode() + sep + str(w).encode() + sep + str(h).encode()
        if kind in "25":
            head += sep + b"255"
        if kind == "1":
            vals = rng.integers(0, 2, size=w * h)
            body = b"".join((b"%d" % v) + (b" " if rng.random() < 0.5 else b"") for v in vals)
            out.append(head + b"\n" + body)
        elif kind == "2":
            vals = rng.integers(0, 256, size=w * h)
            out.append(head + b"\n" + b" ".join(b"%d" % v for v in vals) + b"\n")
        elif kind == "4":
            stride = (w + 7) // 8
            out.append(head + b"\n" + rng.integers(0, 256, size=stride * h, dtype=np.uint8).tobytes())
        else:
            out.append(head + b"\n" + rng.integers(0, 256, size=w * h, dtype=np.uint8).tobytes())
    return out


def broken_files(rng: np.random.Generator, good: list[bytes]) -> list[bytes]:
    out = [b"", b"P", b"Q4\n1 1\n", b"P9\n1 1\n", b"P1\n2\n", b"P1\n2 2\n1 0 0\n", b"P1\n2 2\n1 0 0 2\n",
           b"P5 2 2 255\n\x01\x02", b"P3\n1 1\n255\n0 0 0\n", b"P6\n1 1\n255\n", b"P7\n", b"P5\n1 1\n65535\n",
           b"P2\n1 1\n15\n0\n", b"P2\n1 1\n255\n300\n", b"P4\n3 1\n", b"P4\n3 1\nX", b"P4 3 1", b"P1 99999999999 1\n",
           b"P2\n2 1\n255\n12 a\n", b"P4\n#c\n8 1\n\xff", b"P4\n8 2\n\xff"]
    for f in good[:60]:
        if len(f) > 3:
            cut = int(rng.integers(1, len(f)))
            out.append(f[:cut])
            b = bytearray(f)
            b[int(rng.integers(0, min(len(b), 12)))] = int(rng.integers(0, 256))
            out.append(bytes(b))
    return out
