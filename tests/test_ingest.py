"""PGM/PPM ingest (proj/src/image.cpp:17-92): the C-ABI
header parser against the reference's own load_image tests
(proj/tests/test_image.cpp:34-85), and the oracle's P6 grey conversion.
CPU only: the parser is host code in the extractor library."""
import numpy as np
import pytest

import oracle_lib
import paper_1705_09776_b200 as cg


def pnm(header: bytes, raster: bytes) -> bytes:
    return header + raster


def test_pgm_header_and_raster_offset():
    # test_image.cpp:34-47 ("pgm bytes scale linearly by 1/255")
    raster = bytes([0, 255, 128, 64] + [0] * 60)
    data = pnm(b"P5\n8 8\n255\n", raster)
    w, h, ch, off = cg.parse_pnm(data)
    assert (w, h, ch) == (8, 8, 1)
    assert data[off:off + 4] == bytes([0, 255, 128, 64])


def test_ppm_header_comments_and_whitespace():
    raster = bytes(range(256)) * 3  # 16 x 16 x 3 = 768 bytes
    data = pnm(b"P6 # colour\n# comment line\n16\t16  # trailing\n255 ", raster)
    w, h, ch, off = cg.parse_pnm(data)
    assert (w, h, ch) == (16, 16, 3)
    assert data[off:] == raster


@pytest.mark.parametrize("data", [
    b"P9\n8 8\n255\n" + bytes(64),            # test_image.cpp:68-72 unsupported magic
    b"P5\n2 2\n255\n" + bytes(4),             # :74-78 below 8 px per side
    b"P5\n8 8\n65535\n" + bytes(128),         # :80-85 maxval other than 255
    b"P5\n8 8\n255\n" + bytes(63),            # truncated raster
    b"P6\n8 8\n255\n" + bytes(64 * 3 - 1),    # truncated colour raster
    b"P5\n8 x\n255\n" + bytes(64),            # invalid header field
    b"P5\n8 -8\n255\n" + bytes(64),           # negative field
    b"P5\n8",                                 # truncated header
    b"",
])
def test_malformed_files_raise_data_error(data):
    with pytest.raises(cg.DataError):
        cg.parse_pnm(data)


def test_oracle_ppm_grey_weights():
    # test_image.cpp:49-66: white -> 1, pure red -> 0.299 (exact double expression)
    white = np.full((8, 8, 3), 255, dtype=np.uint8)
    g = oracle_lib.grey_rgb(white)
    assert g.max() <= 1.0 and g[3, 3] == pytest.approx(1.0)
    red = np.zeros((8, 8, 3), dtype=np.uint8)
    red[0, 0, 0] = 255
    g = oracle_lib.grey_rgb(red)
    assert g[0, 0] == (0.299 * 255 + 0.587 * 0 + 0.114 * 0) * (1.0 / 255.0)
    assert g[0, 0] == pytest.approx(0.299, rel=1e-6)
    rng = np.random.default_rng(7)
    px = rng.integers(0, 256, size=(9, 11, 3), dtype=np.uint8)
    want = (0.299 * px[..., 0].astype(np.float64) + 0.587 * px[..., 1] + 0.114 * px[..., 2]) * (1.0 / 255.0)
    assert np.array_equal(oracle_lib.grey_rgb(px), want)
