"""PLY ingestion (reference src/ply.cpp:53-225, tests test_scene.cpp:44-125).

Header parsing and ASCII bodies run on the host and are checked here on CPU against the
reference's own load_ply (oracle/_ref/libgss_ref.so): identical values bit for bit, identical
ParseError messages. Binary bodies are decoded by a kernel (gpu tests): identical values vs the
reference for every scalar type, preceding elements, truncation and non-finite vertices, a 2M-
vertex file, and the PLY -> init_gaussians path vs the reference's init_gaussians.
"""
import struct

import numpy as np
import pytest

import oracles as O
import paper_2509_15645_b200 as G

HDR = "ply\nformat {fmt} 1.0\n"


def write(path, text, body=b""):
    with open(path, "wb") as f:
        f.write(text.encode() if isinstance(text, str) else text)
        f.write(body)
    return path


def ours(path, device=None):
    try:
        pc = G.load_ply(path, device=device)
    except G.ParseError as e:
        return "ParseError: " + str(e).split("] ", 1)[1]
    pos = pc.positions if device is None else pc.positions.cpu().numpy()
    col = pc.colors if (device is None or pc.colors is None) else pc.colors.cpu().numpy()
    return pos, col


def theirs(path):
    try:
        return O.ref_load_ply(path)
    except RuntimeError as e:
        return str(e)


def same(a, b):
    if isinstance(a, str) or isinstance(b, str):
        assert a == b
        return
    assert np.array_equal(a[0].view(np.uint32), b[0].view(np.uint32))
    assert (a[1] is None) == (b[1] is None)
    if a[1] is not None:
        assert np.array_equal(a[1].view(np.uint32), b[1].view(np.uint32))


ASCII_CASES = {
    # test_scene.cpp:44-54
    "tri": HDR + "element vertex 3\nproperty float x\nproperty float y\nproperty float z\nend_header\n"
                 "0 0 0\n1 0 0\n0 1 0\n",
    # test_scene.cpp:56-68
    "uchar_colour": HDR + "element vertex 1\nproperty float x\nproperty float y\nproperty float z\n"
                          "property uchar red\nproperty uchar green\nproperty uchar blue\nend_header\n"
                          "1 2 3 255 0 51\n",
    "float_colour_clamped": HDR + "element vertex 2\nproperty double x\nproperty double y\nproperty double z\n"
                                  "property float r\nproperty float g\nproperty float b\nend_header\n"
                                  "0.1 0.2 0.3 -0.5 0.25 7\n1e-3 -2.5e10 3.14159265358979 0.5 nan 1\n",
    # test_scene.cpp:70-81
    "missing_z": HDR + "element vertex 1\nproperty float x\nproperty float y\nend_header\n1 2\n",
    # test_scene.cpp:83-94
    "bad_keyword": "ply\nformat ascii 1.0\nelemnt vertex 1\nend_header\n",
    # test_scene.cpp:96-108
    "nan_vertex": HDR + "element vertex 2\nproperty float x\nproperty float y\nproperty float z\nend_header\n"
                        "1 2 3\n1 nan 3\n",
    "inf_vertex": HDR + "element vertex 3\nproperty float x\nproperty float y\nproperty float z\nend_header\n"
                        "1 2 3\n4 5 6\ninf 1 1\n",
    "no_magic": "plx\nformat ascii 1.0\n",
    "no_format": "ply\nelement vertex 1\nproperty float x\nproperty float y\nproperty float z\nend_header\n1 2 3\n",
    "bad_format": "ply\nformat binary_big_endian 1.0\nelement vertex 1\nend_header\n",
    "no_vertex": HDR + "element face 1\nproperty list uchar int vertex_indices\nend_header\n3 0 1 2\n",
    "empty_vertex": HDR + "element vertex 0\nproperty float x\nproperty float y\nproperty float z\nend_header\n",
    "bad_element": HDR + "element vertex -4\nend_header\n",
    "prop_first": HDR + "property float x\nelement vertex 1\nend_header\n",
    "bad_prop_type": HDR + "element vertex 1\nproperty float128 x\nend_header\n",
    "bad_list": HDR + "element vertex 1\nproperty list uchar foo idx\nend_header\n",
    "header_eof": HDR + "element vertex 1\nproperty float x\n",
    "truncated": HDR + "element vertex 3\nproperty float x\nproperty float y\nproperty float z\nend_header\n1 2 3\n",
    "short_row": HDR + "element vertex 1\nproperty float x\nproperty float y\nproperty float z\nend_header\n1 2\n",
    "bad_token": HDR + "element vertex 1\nproperty float x\nproperty float y\nproperty float z\nend_header\n1 q 3\n",
    "blank_lines_crlf_comments": "ply\r\nformat ascii 1.0\r\ncomment made by hand\r\nobj_info x\r\n"
                                 "element vertex 2\r\nproperty float x\r\nproperty float y\r\nproperty float z\r\n"
                                 "end_header\r\n\r\n  \r\n1.5 -2 3e2\r\n\t\n0x10 1e-45 -0\r\n",
    "elements_before_vertex": HDR + "element camera 2\nproperty float a\nproperty int b\n"
                                    "element vertex 2\nproperty float x\nproperty float y\nproperty float z\n"
                                    "property uchar red\nproperty uchar green\nproperty uchar blue\n"
                                    "element face 1\nproperty list uchar int vertex_indices\nend_header\n"
                                    "1 2\n3 4\n0.5 0.25 0.125 10 20 30\n1 1 1 0 0 255\n3 0 1 1\n",
    "list_before_vertex": HDR + "element face 1\nproperty list uchar int idx\n"
                                "element vertex 1\nproperty float x\nproperty float y\nproperty float z\n"
                                "end_header\n3 0 1 2\n1 2 3\n",
    "extra_props": HDR + "element vertex 2\nproperty float nx\nproperty float x\nproperty float ny\n"
                         "property float y\nproperty float z\nproperty float opacity\nend_header\n"
                         "9 1 9 2 3 0.5\n9 4 9 5 6 0.5\n",
}


@pytest.mark.parametrize("name", sorted(ASCII_CASES))
def test_ascii_and_header_vs_reference(tmp_path, ref, name):
    p = write(tmp_path / f"{name}.ply", ASCII_CASES[name].format(fmt="ascii"))
    same(ours(p), theirs(p))


def test_missing_file(tmp_path, ref):
    p = tmp_path / "nope.ply"
    same(ours(p), theirs(p))


def test_save_ply_bytes_equal_reference(tmp_path, ref):
    rng = np.random.default_rng(3)
    pos = rng.normal(size=(50, 3)).astype(np.float32)
    col = rng.uniform(-0.1, 1.1, size=(50, 3)).astype(np.float32)
    for binary in (True, False):
        for c in (col, None):
            G.save_ply(tmp_path / "a.ply", G.PointCloud(pos, c), binary=binary)
            O.ref_save_ply(tmp_path / "b.ply", pos, c, binary=binary)
            assert (tmp_path / "a.ply").read_bytes() == (tmp_path / "b.ply").read_bytes()


# ---- binary bodies: device decode --------------------------------------------------------

FMT = {"uchar": "B", "char": "b", "ushort": "H", "short": "h", "uint": "I", "int": "i", "float": "f",
       "double": "d", "uint8": "B", "int16": "h", "float32": "f", "float64": "d"}


def binary_file(path, props, rows, pre=None, truncate=0):
    """props: [(type, name)], rows: list of tuples; pre: (name, props, rows) element before vertex."""
    h = "ply\nformat binary_little_endian 1.0\n"
    body = b""
    if pre:
        h += f"element {pre[0]} {len(pre[2])}\n" + "".join(f"property {t} {n}\n" for t, n in pre[1])
        body += b"".join(struct.pack("<" + "".join(FMT[t] for t, _ in pre[1]), *r) for r in pre[2])
    h += f"element vertex {len(rows)}\n" + "".join(f"property {t} {n}\n" for t, n in props) + "end_header\n"
    body += b"".join(struct.pack("<" + "".join(FMT[t] for t, _ in props), *r) for r in rows)
    if truncate:
        body = body[:-truncate]
    return write(path, h, body)


BIN_CASES = {
    "float_uchar": ([("float", "x"), ("float", "y"), ("float", "z"), ("uchar", "red"), ("uchar", "green"),
                     ("uchar", "blue")], [(0.5, -1.0, 2.0, 0, 128, 255), (1e30, -1e-30, 3.0, 7, 8, 9)], None, 0),
    "double_mixed_colour": ([("double", "x"), ("short", "q"), ("double", "y"), ("double", "z"), ("float", "r"),
                             ("char", "g"), ("ushort", "b")],
                            [(0.1, -3, 0.2, 0.3, 1.5, -5, 300), (1e300, 0, -2.0, 5.0, -0.25, 127, 0)], None, 0),
    "ints": ([("int", "x"), ("uint", "y"), ("int16", "z")], [(-7, 4000000000, -32768), (2147483647, 0, 5)], None, 0),
    "pre_element": ([("float", "x"), ("float", "y"), ("float", "z")], [(1, 2, 3), (4, 5, 6)],
                    ("camera", [("float", "a"), ("double", "b")], [(1.0, 2.0), (3.0, 4.0), (5.0, 6.0)]), 0),
    "truncated": ([("float", "x"), ("float", "y"), ("float", "z")], [(1, 2, 3), (4, 5, 6), (7, 8, 9)], None, 5),
    "truncated_pre": ([("float", "x"), ("float", "y"), ("float", "z")], [(1, 2, 3)],
                      ("camera", [("float", "a")], [(1.0,), (2.0,), (3.0,)]), 14),
    "nonfinite": ([("float", "x"), ("float", "y"), ("float", "z")],
                  [(1, 2, 3), (4, 5, 6), (7, float("inf"), 9), (float("nan"), 0, 0)], None, 0),
}


@pytest.mark.gpu
@pytest.mark.parametrize("name", sorted(BIN_CASES))
def test_binary_decode_vs_reference(tmp_path, ref, name):
    props, rows, pre, tr = BIN_CASES[name]
    p = binary_file(tmp_path / f"{name}.ply", props, rows, pre, tr)
    same(ours(p), theirs(p))


@pytest.mark.gpu
def test_binary_large_file_to_device_vs_reference(tmp_path, ref):
    import torch

    rng = np.random.default_rng(11)
    m = 2_000_000
    pos = rng.normal(scale=50.0, size=(m, 3)).astype(np.float32)
    col = rng.uniform(0, 1, size=(m, 3)).astype(np.float32)
    p = tmp_path / "big.ply"
    O.ref_save_ply(p, pos, col, binary=True)  # the reference writer (uchar colours)
    want = theirs(p)
    same(ours(p), want)
    same(ours(p, device=torch.device("cuda")), want)


@pytest.mark.gpu
def test_ply_to_init_gaussians_vs_reference(tmp_path, ref):
    rng = np.random.default_rng(5)
    m = 3000
    pos = rng.uniform(-1, 1, size=(m, 3)).astype(np.float32)
    col = rng.uniform(0, 1, size=(m, 3)).astype(np.float32)
    p = tmp_path / "scene.ply"
    O.ref_save_ply(p, pos, col, binary=True)
    rows = G.init_from_ply(p)
    rp, rc = O.ref_load_ply(p)
    want = np.zeros((m, 59), np.float32)
    assert O.ref().ref_init_gaussians(rp.ctypes.data, rc.ctypes.data, m, 3, 0.01, 0.1, want.ctypes.data) == 0
    assert np.array_equal(rows.view(np.uint32), want.view(np.uint32))
