"""File I/O of the framework: load_image / save_pgm (image_io.cpp:19-160) and
the .flo reader/writer (metrics.cpp:22-73). Host-side formats, so these run without a GPU.
PNG files are written here by a small encoder that exercises every filter type, bit depth
and colour type the loader accepts; .flo bytes are compared with the reference's writer."""
import struct
import zlib

import numpy as np
import pytest

from paper_1508_02977_b200 import flowfem as ff


def _chunk(t, d):
    return struct.pack(">I", len(d)) + t + d + struct.pack(">I", zlib.crc32(t + d) & 0xffffffff)


def _paeth(a, b, c):
    p = a + b - c
    pa, pb, pc = abs(p - a), abs(p - b), abs(p - c)
    return a if pa <= pb and pa <= pc else (b if pb <= pc else c)


def write_png(path, rows_bytes, W, H, depth, color, bpp, palette=None, trns=None):
    """rows_bytes: H raw scanlines (unfiltered); filter type = row index % 5."""
    raw = b""
    prev = bytes(len(rows_bytes[0]))
    for y, row in enumerate(rows_bytes):
        ft = y % 5
        out = bytearray()
        for i, v in enumerate(row):
            a = row[i - bpp] if i >= bpp else 0
            b = prev[i]
            c = prev[i - bpp] if i >= bpp else 0
            pred = [0, a, b, (a + b) >> 1, _paeth(a, b, c)][ft]
            out.append((v - pred) & 0xff)
        raw += bytes([ft]) + bytes(out)
        prev = row
    data = b"\x89PNG\r\n\x1a\n" + _chunk(b"IHDR", struct.pack(">IIBBBBB", W, H, depth, color, 0, 0, 0))
    if palette is not None:
        data += _chunk(b"PLTE", bytes(palette))
    if trns is not None:
        data += _chunk(b"tRNS", bytes(trns))
    z = zlib.compress(raw)
    data += _chunk(b"IDAT", z[:len(z) // 2]) + _chunk(b"IDAT", z[len(z) // 2:]) + _chunk(b"IEND", b"")
    with open(path, "wb") as f:
        f.write(data)


def pack_bits(vals, depth):
    out = bytearray()
    acc, nb = 0, 0
    for v in vals:
        acc = (acc << depth) | int(v)
        nb += depth
        if nb == 8:
            out.append(acc)
            acc, nb = 0, 0
    if nb:
        out.append(acc << (8 - nb))
    return bytes(out)


RGBW = np.array([0.299, 0.587, 0.114])


@pytest.mark.parametrize("depth", [8, 16])
def test_png_gray(tmp_path, depth):
    rng = np.random.default_rng(depth)
    H, W = 11, 13
    mx = (1 << depth) - 1
    img = rng.integers(0, mx + 1, (H, W))
    rows = [b"".join(int(v).to_bytes(depth // 8, "big") for v in r) for r in img]
    write_png(tmp_path / "g.png", rows, W, H, depth, 0, depth // 8)
    assert np.array_equal(ff.load_image(str(tmp_path / "g.png")), img / float(mx))


@pytest.mark.parametrize("depth", [1, 2, 4])
def test_png_low_bit_gray_expanded(tmp_path, depth):
    rng = np.random.default_rng(depth)
    H, W = 7, 19
    img = rng.integers(0, 1 << depth, (H, W))
    rows = [pack_bits(r, depth) for r in img]
    write_png(tmp_path / "g.png", rows, W, H, depth, 0, 1)
    expect = (img * 255 // ((1 << depth) - 1)) / 255.0
    assert np.array_equal(ff.load_image(str(tmp_path / "g.png")), expect)


@pytest.mark.parametrize("color,depth", [(2, 8), (6, 8), (2, 16), (6, 16), (4, 8)])
def test_png_color_and_alpha(tmp_path, color, depth):
    rng = np.random.default_rng(color * 100 + depth)
    H, W = 9, 10
    ch = {2: 3, 6: 4, 4: 2}[color]
    mx = (1 << depth) - 1
    img = rng.integers(0, mx + 1, (H, W, ch))
    nb = depth // 8
    rows = [b"".join(int(v).to_bytes(nb, "big") for v in r.ravel()) for r in img]
    write_png(tmp_path / "c.png", rows, W, H, depth, color, ch * nb)
    got = ff.load_image(str(tmp_path / "c.png"))
    if ch >= 3:
        s = img[..., :3] / float(mx)
        expect = 0.299 * s[..., 0] + 0.587 * s[..., 1] + 0.114 * s[..., 2]
    else:
        expect = img[..., 0] / float(mx)
    assert np.array_equal(got, expect)


@pytest.mark.parametrize("depth", [8, 4])
def test_png_palette(tmp_path, depth):
    rng = np.random.default_rng(depth)
    H, W = 6, 15
    ncol = 1 << depth if depth < 8 else 200
    pal = rng.integers(0, 256, (ncol, 3))
    idx = rng.integers(0, ncol, (H, W))
    rows = [pack_bits(r, depth) if depth < 8 else bytes(int(v) for v in r) for r in idx]
    write_png(tmp_path / "p.png", rows, W, H, depth, 3, 1, palette=pal.ravel().tolist(),
              trns=[128] * 3)
    s = pal[idx] / 255.0
    expect = 0.299 * s[..., 0] + 0.587 * s[..., 1] + 0.114 * s[..., 2]
    assert np.array_equal(ff.load_image(str(tmp_path / "p.png")), expect)


def test_pgm_8_and_16_bit_with_comments(tmp_path):
    rng = np.random.default_rng(0)
    img = rng.integers(0, 256, (5, 7))
    (tmp_path / "a.pgm").write_bytes(b"P5\n# a comment\n7 5\n# another\n255\n" + bytes(img.astype(np.uint8).ravel()))
    assert np.array_equal(ff.load_image(str(tmp_path / "a.pgm")), img / 255.0)
    img16 = rng.integers(0, 1001, (4, 3))
    (tmp_path / "b.pgm").write_bytes(b"P5 3 4 1000\n" + img16.astype(">u2").tobytes())
    assert np.array_equal(ff.load_image(str(tmp_path / "b.pgm")), img16 / 1000.0)


def test_image_errors(tmp_path):
    (tmp_path / "t.pgm").write_bytes(b"P5\n7 5\n255\n" + bytes(10))
    with pytest.raises(ff.FlowfemError, match="imaging.load_image: truncated PGM data"):
        ff.load_image(str(tmp_path / "t.pgm"))
    (tmp_path / "a.txt").write_bytes(b"P2\n1 1\n255\n0\n")
    with pytest.raises(ff.FlowfemError, match=r"unrecognized format \(want PGM P5 or PNG\)"):
        ff.load_image(str(tmp_path / "a.txt"))
    with pytest.raises(ff.FlowfemError, match="imaging.load_image: cannot open"):
        ff.load_image(str(tmp_path / "missing.png"))
    (tmp_path / "z.pgm").write_bytes(b"P5\n0 5\n255\n")
    with pytest.raises(ff.FlowfemError, match="bad PGM dimensions"):
        ff.load_image(str(tmp_path / "z.pgm"))


def test_save_pgm_roundtrip(tmp_path):
    img = np.array([[-0.5, 0.0, 0.5, 1.0, 2.0], [0.3, 0.7, 1 / 255, 0.998, 0.002]])
    ff.save_pgm(str(tmp_path / "o.pgm"), img)
    data = (tmp_path / "o.pgm").read_bytes()
    assert data.startswith(b"P5\n5 2\n255\n")
    expect = (np.clip(img, 0, 1) * 255.0 + 0.5).astype(np.uint8)
    assert data[len(b"P5\n5 2\n255\n"):] == bytes(expect.ravel())
    assert np.array_equal(ff.load_image(str(tmp_path / "o.pgm")), expect / 255.0)


def test_flo_roundtrip_and_reference_bytes(tmp_path, ref):
    import pyoracle as po
    rng = np.random.default_rng(5)
    u = rng.normal(size=(6, 9)).astype(np.float32)
    v = rng.normal(size=(6, 9)).astype(np.float32)
    v[2, 3] = 1e10
    ff.write_flo(str(tmp_path / "a.flo"), ff.FloField(u, v))
    po.ref_write_flo(str(tmp_path / "r.flo"), u, v)
    assert (tmp_path / "a.flo").read_bytes() == (tmp_path / "r.flo").read_bytes()
    f = ff.read_flo(str(tmp_path / "r.flo"))
    assert np.array_equal(f.u, u) and np.array_equal(f.v, v) and (f.width, f.height) == (9, 6)
    flow = rng.normal(size=(3, 6, 9))
    tu, tv = po.ref_to_flo(flow)
    mine = ff.to_flo(ff.FlowState.from_planes(flow))
    assert np.array_equal(mine.u, tu) and np.array_equal(mine.v, tv)


def test_flo_errors(tmp_path):
    (tmp_path / "b.flo").write_bytes(struct.pack("<fii", 1.0, 2, 2) + bytes(32))
    with pytest.raises(ff.FlowfemError, match="metrics.read_flo: bad magic"):
        ff.read_flo(str(tmp_path / "b.flo"))
    (tmp_path / "t.flo").write_bytes(struct.pack("<fii", 202021.25, 2, 2) + bytes(8))
    with pytest.raises(ff.FlowfemError, match="metrics.read_flo: truncated data"):
        ff.read_flo(str(tmp_path / "t.flo"))
    (tmp_path / "d.flo").write_bytes(struct.pack("<fii", 202021.25, 0, 2))
    with pytest.raises(ff.FlowfemError, match="metrics.read_flo: implausible dimensions"):
        ff.read_flo(str(tmp_path / "d.flo"))
