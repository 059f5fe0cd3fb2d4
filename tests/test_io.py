"""io formats either side of the stereo path (SPEC.md
[MODULE] io :517-534 and run_stereo_only :581-589). The reference has no io
source; the SPEC's examples are the fixtures. Host parts run on CPU through
tests/cpp/io_tool (include/stereoscan/io/io.hpp); run_stereo_only drives the
GPU path (-m gpu).
"""
import os
import struct
import subprocess
import zlib

import numpy as np
import pytest

from conftest import ROOT

TOOL = os.path.join(ROOT, "tests", "cpp", "build", "io_tool")


@pytest.fixture(scope="module")
def tool():
    from paper_2007_12623_b200.build import build
    build(verbose=False)
    assert os.path.exists(TOOL)

    def run(*args):
        r = subprocess.run([TOOL, *map(str, args)], capture_output=True, text=True, timeout=600)
        assert r.returncode == 0, r.stderr
        return r.stdout.strip()
    return run


def png_bytes(img, filt):
    """Independent PNG encoder: 8-bit grey / RGB / RGBA, one filter type per row."""
    h, w = img.shape[:2]
    ch = 1 if img.ndim == 2 else img.shape[2]
    ctype = {1: 0, 2: 4, 3: 2, 4: 6}[ch]
    a = img.reshape(h, w * ch).astype(np.int32)
    raw = bytearray()
    for y in range(h):
        cur, up = a[y], a[y - 1] if y else np.zeros_like(a[y])
        left = np.concatenate([np.zeros(ch, np.int32), cur[:-ch]])
        ul = np.concatenate([np.zeros(ch, np.int32), up[:-ch]])
        if filt == 0:
            pred = np.zeros_like(cur)
        elif filt == 1:
            pred = left
        elif filt == 2:
            pred = up
        elif filt == 3:
            pred = (left + up) // 2
        else:
            p = left + up - ul
            pa, pb, pc = abs(p - left), abs(p - up), abs(p - ul)
            pred = np.where((pa <= pb) & (pa <= pc), left, np.where(pb <= pc, up, ul))
        raw.append(filt)
        raw += bytes(((cur - pred) & 0xFF).astype(np.uint8))

    def chunk(t, d):
        return struct.pack(">I", len(d)) + t + d + struct.pack(">I", zlib.crc32(t + d) & 0xFFFFFFFF)
    return (b"\x89PNG\r\n\x1a\n" + chunk(b"IHDR", struct.pack(">IIBBBBB", w, h, 8, ctype, 0, 0, 0))
            + chunk(b"IDAT", zlib.compress(bytes(raw))) + chunk(b"IEND", b""))


def rgb_of(img):
    if img.ndim == 2:
        return np.repeat(img[:, :, None], 3, 2)
    if img.shape[2] == 2:
        return np.repeat(img[:, :, :1], 3, 2)
    return img[:, :, :3]


@pytest.mark.parametrize("ch", [1, 2, 3, 4])
@pytest.mark.parametrize("filt", [0, 1, 2, 3, 4])
def test_png_decode(tool, tmp_path, ch, filt):
    rng = np.random.default_rng(ch * 10 + filt)
    img = rng.integers(0, 256, (13, 17, ch) if ch > 1 else (13, 17), dtype=np.uint8)
    p = tmp_path / "x.png"
    p.write_bytes(png_bytes(img, filt))
    w, h, s = tool("png", p).split()
    assert (int(w), int(h)) == (17, 13) and int(s) == int(rgb_of(img).astype(np.int64).sum())


def test_png_save_roundtrip_and_errors(tool, tmp_path):
    p = tmp_path / "g.png"
    tool("pngsave", p, 5, 3)
    expect = sum((i * 7) % 251 for i in range(45))
    assert tool("png", p) == f"5 3 {expect}"
    b1 = p.read_bytes()
    tool("pngsave", p, 5, 3)
    assert p.read_bytes() == b1  # deterministic bytes
    bad = tmp_path / "bad.png"
    bad.write_bytes(b"not a png")
    assert tool("png", bad).startswith("ERROR") and "not a PNG" in tool("png", bad)
    assert "cannot open" in tool("png", tmp_path / "missing.png")


CAL = "fx = 1000\nfy=1000\ncx = 480  # comment\ncy = 270\nbaseline_mm = 5\nwidth = 960\nheight = 540\n"


def test_calibration(tool, tmp_path):
    p = tmp_path / "c.txt"
    p.write_text(CAL)
    assert tool("calib", p).split() == ["1000", "1000", "480", "270", "960", "540", "5"]
    p.write_text(CAL.replace("baseline_mm = 5", "baseline_mm = -1"))
    out = tool("calib", p)
    assert out.startswith("ERROR") and "baseline" in out
    p.write_text(CAL.replace("fy=1000\n", ""))
    out = tool("calib", p)
    assert out.startswith("ERROR") and '"fy"' in out
    p.write_text(CAL.replace("fx = 1000", "fx = abc"))
    out = tool("calib", p)
    assert out.startswith("ERROR") and ":1:" in out and '"fx"' in out
    p.write_text(CAL + "gamma = 2\n")
    assert "unknown key" in tool("calib", p)


def test_pgm16(tool, tmp_path):
    p = tmp_path / "d.pgm"
    tool("pgm", p)
    b = p.read_bytes()
    assert b.startswith(b"P5\n4 2\n65535\n")
    v = np.frombuffer(b[len(b"P5\n4 2\n65535\n"):], ">u2")
    # 7 -> 7*256; 7.5 -> 1920; negative -> 0; 300*256 -> clamp 65535;
    # invalid -> 0; 0.001*256 -> 0; 255.998*256 -> 65535.5 -> 65535 (clamped)
    assert v.tolist() == [1792, 1920, 0, 65535, 0, 0, 65535, 0]


def test_ply(tool, tmp_path):
    p = tmp_path / "c.ply"
    tool("ply", p, 0)
    assert b"element vertex 0\n" in p.read_bytes()  # empty model -> valid PLY
    tool("ply", p, 2)
    b = p.read_bytes()
    head, body = b.split(b"end_header\n")
    assert b"format binary_little_endian 1.0" in head and len(body) == 2 * 27
    rec = struct.unpack("<6f3B", body[27:54])
    assert rec == (1.0, 2.0, 3.0, 0.0, 0.0, -1.0, 255, 255, 255)


@pytest.mark.gpu
def test_run_stereo_only(tool, tmp_path):
    import paper_2007_12623_b200 as ss
    # a 7-px shifted texture -> PGM uniform at 7*256 over the interior
    rng = np.random.default_rng(3)
    tex = rng.integers(0, 256, (64, 200), dtype=np.uint8)
    L, R = tex[:, :160], tex[:, 7:167]
    d = tmp_path / "seq"
    d.mkdir()
    (d / "left_000003.png").write_bytes(png_bytes(np.repeat(L[:, :, None], 3, 2), 4))
    (d / "right_000003.png").write_bytes(png_bytes(np.repeat(R[:, :, None], 3, 2), 1))
    cal = tmp_path / "cal.txt"
    cal.write_text("fx = 500\nfy = 500\ncx = 80\ncy = 32\nbaseline_mm = 5\nwidth = 160\nheight = 64\n")
    out = tool("stereo", cal, d, 3, tmp_path / "f3", 0, 15)
    assert out.startswith("points") and int(out.split()[1]) > 0, out
    b = (tmp_path / "f3_disparity.pgm").read_bytes()
    v = np.frombuffer(b[len(b"P5\n160 64\n65535\n"):], ">u2").reshape(64, 160)
    # the PGM is the full stage's map (the reference's refinement drifts a few
    # hundredths of a pixel near the filled border; the WTA itself is 7 everywhere)
    p = {"d_min": 0, "d_max": 15}
    dw, vw = ss.compute_disparity(L, R, p)
    assert np.all(dw[vw == 1] == 7.0)
    dd, vv = ss.cleanup_pass(dw, vw, p)
    dd, vv = ss.refine_disparities(dd, vv, L, R, p)
    q = np.where(vv == 1, np.clip(np.floor(dd.astype(np.float64) * 256 + 0.5), 0, 65535), 0)
    assert np.array_equal(v, q.astype(np.uint16))
    assert np.median(v[10:-10, 30:-10]) == 7 * 256
    ply = (tmp_path / "f3.ply").read_bytes()
    assert f"element vertex {out.split()[1]}\n".encode() in ply
    # uniform pair -> all zeros
    U = np.full((64, 160, 3), 120, np.uint8)
    (d / "left_000004.png").write_bytes(png_bytes(U, 0))
    (d / "right_000004.png").write_bytes(png_bytes(U, 0))
    tool("stereo", cal, d, 4, tmp_path / "f4", 0, 15)
    b = (tmp_path / "f4_disparity.pgm").read_bytes()
    assert not np.frombuffer(b[len(b"P5\n160 64\n65535\n"):], ">u2").any()
    # missing frame -> error; size mismatch -> error
    assert tool("stereo", cal, d, 9, tmp_path / "f9", 0, 15).startswith("ERROR")
    cal.write_text("fx = 500\nfy = 500\ncx = 80\ncy = 32\nbaseline_mm = 5\nwidth = 100\nheight = 100\n")
    assert "does not match" in tool("stereo", cal, d, 3, tmp_path / "f5", 0, 15)
    # pure red -> gray 76
    assert ss.to_gray(np.array([[[255, 0, 0]]], np.uint8))[0, 0] == 76
