"""Dataset loaders and writers (proj/src/graph_io.cpp:41-296) on CPU:
the product's host readers (libsagecut_cuda.so, graph_io.cpp) against the REFERENCE's own
loaders compiled from its sources (oracle/_ref/ref_io_main), on valid files and on every
rejection rule the reference has — same parsed values, same exception type and message.
Writers: the bytes the reference writes after loading the same file.
"""
import os
import subprocess

import numpy as np
import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
REF_IO = os.path.join(ROOT, "oracle", "_ref", "ref_io_main")
pytestmark = pytest.mark.skipif(not os.path.exists(REF_IO), reason="oracle/_ref not built (needs /root/reference)")


@pytest.fixture(scope="module")
def sc():
    from paper_2308_03209_b200 import sagecut  # host-only entry points: no GPU needed
    return sagecut


def ref(*args):
    out = subprocess.run([REF_IO, *map(str, args)], capture_output=True, timeout=120).stdout.decode()
    return out.split("\n")


def ours(fn):
    try:
        return ("ok", fn())
    except (ValueError, RuntimeError) as e:
        kind = "invalid_argument" if isinstance(e, ValueError) else "runtime_error"
        return ("error", kind, str(e).split(": ", 1)[1])


def check_error(r, o):
    assert r[0].startswith("error"), (r[:2], o)
    kind, msg = r[0].split(" ", 2)[1:]
    assert o[0] == "error" and o[1] == kind and o[2] == msg, (r[0], o)


EDGE_FILES = {
    "plain": "0 1\n1 2\n2 0\n3 4\n",
    "comments_blank_crlf": "# karate-like\n\n  # indented comment\n0 1\r\n1 2\r\n\t2 3\n5 5\n3 2\n",
    "isolated_tail": "0 1\n1 2\n",
    "bad_token": "0 1\n1 x\n",
    "one_token": "0 1\n7\n",
    "trailing": "0 1\n1 2 3\n",
    "negative": "0 1\n-1 2\n",
    "plus_sign": "+0 +1\n",
    "glued": "0 1\n12abc 3\n",
    "float": "0 1\n1.5 2\n",
    "empty": "",
}


@pytest.mark.parametrize("name", sorted(EDGE_FILES))
def test_edge_list(sc, tmp_path, name):
    p = tmp_path / f"{name}.edges"
    p.write_text(EDGE_FILES[name])
    for nn, strict in ((-1, 0), (10, 0), (3, 0)):
        r = ref("graph", p, nn, strict)
        o = ours(lambda: sc.read_edge_list(str(p), None if nn < 0 else nn))
        if r[0].startswith("error"):
            check_error(r, o)
            continue
        assert o[0] == "ok", (r[0], o)
        uv, n = o[1]
        assert int(r[0].split()[1]) == n
        # the reference's lines are the canonical edges after build_graph: compare the sets
        ref_edges = {tuple(map(int, ln.split())) for ln in r[1:] if ln.strip()}
        canon = {(min(u, v), max(u, v)) for u, v in uv.tolist() if u != v}
        assert canon == ref_edges


def test_edge_list_missing_and_strict(sc, tmp_path):
    o = ours(lambda: sc.read_edge_list(str(tmp_path / "nope.edges")))
    check_error(ref("graph", tmp_path / "nope.edges", -1, 0), o)


def features_cases(tmp_path):
    rng = np.random.default_rng(0)
    x = rng.standard_normal((7, 5)).astype(np.float32)
    cases = {}
    cases["csv"] = "\n".join(",".join(repr(float(v)) for v in row) for row in x) + "\n"
    cases["csv_comments_ws"] = "# header\n" + "\n".join(" " + ", ".join(f"{v:.6e}" for v in row) + " \r" for row in x)
    cases["csv_ragged"] = "1,2,3\n4,5\n6,7,8\n" + "1,1,1\n" * 4
    cases["csv_bad"] = "1,2,3\n4,zz,6\n" + "1,1,1\n" * 5
    cases["csv_empty_tok"] = "1,2,\n" + "1,1,1\n" * 6
    cases["csv_inf"] = "1,2,3\n4,inf,6\n" + "1,1,1\n" * 5
    cases["csv_rows"] = "1,2\n3,4\n"
    cases["csv_hex"] = "0x1p3,2\n" + "1,1\n" * 6
    return x, cases


def cfm1(x, rows=None, truncate=0, bad=False):
    import struct
    data = b"CFM1" + struct.pack("<QQ", x.shape[0] if rows is None else rows, x.shape[1])
    y = x.copy()
    if bad:
        y[2, 3] = np.nan
    payload = y.astype("<f4").tobytes()
    return data + (payload[:-truncate] if truncate else payload)


def test_features(sc, tmp_path):
    x, cases = features_cases(tmp_path)
    files = {}
    for k, v in cases.items():
        files[k] = tmp_path / f"{k}.csv"
        files[k].write_text(v)
    for k, v in {"bin": cfm1(x), "bin_rows": cfm1(x, rows=9), "bin_trunc": cfm1(x, truncate=6),
                 "bin_nan": cfm1(x, bad=True), "bin_hdr": b"CFM1\x07\x00"}.items():
        files[k] = tmp_path / f"{k}.bin"
        files[k].write_bytes(v)
    for k, p in sorted(files.items()):
        r = ref("features", p, 7, tmp_path / f"{k}.ref.csv", tmp_path / f"{k}.ref.bin")
        o = ours(lambda: sc.load_features(str(p), 7))
        if r[0].startswith("error"):
            check_error(r, o)
            continue
        assert o[0] == "ok", (k, r[0], o)
        rows, cols = map(int, r[0].split()[1:])
        assert o[1].shape == (rows, cols)
        np.testing.assert_array_equal(o[1].ravel(), np.array([float(v) for v in r[1:] if v.strip()], np.float32), err_msg=k)
        # writers: the reference re-saved what it loaded; ours must write the same bytes
        sc.save_features(o[1], str(tmp_path / f"{k}.our.bin"), binary=True)
        assert (tmp_path / f"{k}.our.bin").read_bytes() == (tmp_path / f"{k}.ref.bin").read_bytes()
        if k.startswith("bin"):  # float32 payload: the CSV text of its doubles matches too
            sc.save_features(o[1], str(tmp_path / f"{k}.our.csv"))
            assert (tmp_path / f"{k}.our.csv").read_bytes() == (tmp_path / f"{k}.ref.csv").read_bytes()


LABEL_FILES = {
    "classes": "0\n3\n1\n1\n# c\n\n2\n0\n4\n",
    "classes_junk": "0\n3 x\n1\n1\n2\n0\n4\n",
    "neg": "0\n-3\n1\n1\n2\n0\n4\n",
    "count": "0\n1\n",
    "multi": "1,0,1\n0,0,0\n1,1,1\n0,1,0\n0,0,1\n1,0,0\n0,1,1\n",
    "multi_trailing_comma": "1,0,1,\n0,0,0,\n1,1,1,\n0,1,0,\n0,0,1,\n1,0,0,\n0,1,1,\n",
    "multi_bad": "1,0,1\n0,2,0\n1,1,1\n0,1,0\n0,0,1\n1,0,0\n0,1,1\n",
    "multi_ragged": "1,0,1\n0,0\n1,1,1\n0,1,0\n0,0,1\n1,0,0\n0,1,1\n",
    "multi_crlf": "1,0,1\r\n0,0,0\r\n1,1,1\r\n0,1,0\r\n0,0,1\r\n1,0,0\r\n0,1,1\r\n",
}


@pytest.mark.parametrize("name", sorted(LABEL_FILES))
def test_labels(sc, tmp_path, name):
    p = tmp_path / f"{name}.txt"
    p.write_text(LABEL_FILES[name])
    r = ref("labels", p, 7, tmp_path / "ref.out")
    o = ours(lambda: sc.load_labels(str(p), 7))
    if r[0].startswith("error"):
        check_error(r, o)
        return
    assert o[0] == "ok", (r[0], o)
    lab, y, nc = o[1]
    ml, rc = map(int, r[0].split()[1:])
    assert nc == rc and (y is not None) == bool(ml)
    vals = np.array([int(v) for v in r[1:] if v.strip()])
    np.testing.assert_array_equal((y.ravel() if ml else lab), vals)
    sc.save_labels(str(tmp_path / "our.out"), labels=lab, targets=y)
    assert (tmp_path / "our.out").read_bytes() == (tmp_path / "ref.out").read_bytes()


MASK_FILES = {
    "ok": "train 0\ntrain 3\n# c\n\nval 1\ntest 2\ntest 6\n",
    "range": "train 0\nval 9\n",
    "dup": "train 0\nval 0\n",
    "tag": "train 0\nvalid 1\n",
    "short": "train\n",
    "neg": "test -1\n",
}


@pytest.mark.parametrize("name", sorted(MASK_FILES))
def test_masks(sc, tmp_path, name):
    p = tmp_path / f"{name}.txt"
    p.write_text(MASK_FILES[name])
    r = ref("masks", p, 7, tmp_path / "ref.out")
    o = ours(lambda: sc.load_masks(str(p), 7))
    if r[0].startswith("error"):
        check_error(r, o)
        return
    assert o[0] == "ok", (r[0], o)
    for line, m in zip(r[1:4], o[1]):
        assert line == "".join(str(int(v)) for v in m)
    sc.save_masks(str(tmp_path / "our.out"), *o[1])
    assert (tmp_path / "our.out").read_bytes() == (tmp_path / "ref.out").read_bytes()


def test_missing_files(sc, tmp_path):
    p = tmp_path / "missing"
    check_error(ref("features", p, 7), ours(lambda: sc.load_features(str(p), 7)))
    check_error(ref("labels", p, 7), ours(lambda: sc.load_labels(str(p), 7)))
    check_error(ref("masks", p, 7), ours(lambda: sc.load_masks(str(p), 7)))
