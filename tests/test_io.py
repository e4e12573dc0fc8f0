"""Tensor files: the native parallel .tns reader and
writer, the binary GCPBCOO1 format and the dense raw format, against the
reference's own read_tns / write_tns / read_dense / write_dense
(src/io.cpp:75-250) compiled in oracle/_ref.

Host-only (the readers are CPU code in libgcpb.so): runs under -m "not gpu".
Parity bar: entries, shapes and error messages (including path:line)
identical to the reference; the file-order entry list normalised by the
pinned oracle (or_sparse_normalize, tensor.cpp:10-41) equals the reference's
SparseTensor."""
import numpy as np
import pytest

import oracle as O


def IO():
    import paper_1906_01687_b200.io as io
    return io


def G():
    import paper_1906_01687_b200.gcp as g
    return g


def _normalised(dims, coords, values):
    t = O.Tensor(dims, coords, values)
    return t.coords, t.values


def _assert_same_tensor(ours, ref_tensor):
    assert tuple(ours.dims) == tuple(int(n) for n in ref_tensor.dims)
    rc, rv = ref_tensor.export()
    oc, ov = _normalised(ours.dims, ours.coords, ours.values)
    assert np.array_equal(oc, rc)
    assert np.array_equal(ov, rv)  # bit-exact: same strtod, same summation order


def _errors(ref, path):
    """(our class name, our message), (reference code, reference message)."""
    g = G()
    with pytest.raises(g.GcpError) as ours:
        IO().read_tns(path)
    with pytest.raises(O.RefError) as theirs:
        ref.read_tns(path)
    return ours.value, theirs.value


def _msg(e):
    return str(e.args[0]) if not isinstance(e, O.RefError) else str(e).split("] ", 1)[1]


def test_roundtrip_reference_writer(ref, tmp_path):
    rs = np.random.default_rng(3)
    dims = (13, 7, 9, 5)
    n = 400
    coords = np.stack([rs.integers(0, k, n) for k in dims], 1)
    values = rs.normal(size=n) * 10.0 ** rs.integers(-20, 20, n)
    rt = ref.sparse(dims, coords, values)
    p = tmp_path / "a.tns"
    rt.write_tns(p)
    ours = IO().read_tns(p)
    _assert_same_tensor(ours, rt)
    # our writer -> the reference's reader: identical tensor, %.17g round trip
    q = tmp_path / "b.tns"
    oc, ov = rt.export()
    IO().write_tns(IO().CooTensor(dims, oc, ov), q)
    assert q.read_bytes() == p.read_bytes()
    _assert_same_tensor(IO().read_tns(q), ref.read_tns(q))


def test_format_details_match_reference(ref, tmp_path):
    text = ("# a comment\n"
            "\n"
            "   \t\n"
            "  # indented comment\n"
            "1 2 3 1.5\n"
            "2\t1 1   -2e-3\r\n"
            "1 2 3 0.5\n"          # duplicate: summed
            "3 3 1 0\n"            # explicit zero: dropped
            "+2 01 4 0x1p-3\n"     # strtoll / strtod forms
            "1 1 1 inf\n"
            "3 1 2 1e400")         # no trailing newline; overflow -> inf like strtod
    p = tmp_path / "t.tns"
    p.write_text(text)
    ours = IO().read_tns(p)
    rt = ref.read_tns(p)
    assert ours.dims == (3, 3, 4)  # maxima, no header
    _assert_same_tensor(ours, rt)
    assert ours.nnz == 7  # file order, not normalised


def test_header_and_empty_tensor(ref, tmp_path):
    p = tmp_path / "h.tns"
    p.write_text("#shape: 10 20 30\n# nothing else\n")
    ours = IO().read_tns(p)
    assert ours.dims == (10, 20, 30) and ours.nnz == 0
    assert tuple(ref.read_tns(p).dims) == (10, 20, 30)
    p.write_text("#shape: 10 20 30\n5 5 5 2.0\n")
    _assert_same_tensor(IO().read_tns(p), ref.read_tns(p))


@pytest.mark.parametrize("name,text", [
    ("exceeds", "#shape: 4 4\n1 1 1.0\n5 1 2.0\n"),
    ("zero_index", "1 1 1.0\n0 2 1.0\n"),
    ("bad_int", "1 1 1.0\n1 x 1.0\n"),
    ("bad_float", "1 1 1.0\n1 2 1.0q\n"),
    ("token_count", "1 1 1.0\n1 2 3 1.0\n"),
    ("single_token", "# c\n7\n"),
    ("empty_header", "#shape:   \n1 1 1\n"),
    ("header_zero", "#shape: 3 0\n"),
    ("header_bad", "#shape: 3 a\n"),
    ("empty_file", ""),
    ("only_comments", "# nothing\n\n"),
    ("int_overflow", "99999999999999999999 1 1.0\n"),
    ("vertical_tab_line", "1 1 1.0\n\v\n"),
])
def test_errors_match_reference(ref, tmp_path, name, text):
    p = tmp_path / f"{name}.tns"
    p.write_text(text)
    ours, theirs = _errors(ref, p)
    assert _msg(ours) == _msg(theirs)
    assert type(ours).__name__ == "GcpRuntimeError" and theirs.code == 1


def test_missing_file_matches_reference(ref, tmp_path):
    ours, theirs = _errors(ref, tmp_path / "nope.tns")
    assert _msg(ours) == _msg(theirs)


def test_late_and_repeated_headers_follow_reference(ref, tmp_path):
    # a header after data switches to the exact serial walk
    p = tmp_path / "late.tns"
    p.write_text("1 2 1.0\n#shape: 5 6\n3 6 2.0\n")
    _assert_same_tensor(IO().read_tns(p), ref.read_tns(p))
    # entries before a later header are checked by the tensor constructor
    p.write_text("4 2 1.0\n#shape: 3 6\n")
    g = G()
    with pytest.raises(g.OutOfRange) as ours:
        IO().read_tns(p)
    with pytest.raises(O.RefError) as theirs:
        ref.read_tns(p)
    assert theirs.value.code == 4 and _msg(ours.value) == _msg(theirs.value)
    # headers accumulate: two 1-mode headers declare a 2-mode shape
    p.write_text("#shape: 4\n#shape: 5\n2 3 1.5\n")
    _assert_same_tensor(IO().read_tns(p), ref.read_tns(p))


def _big_text(rs, dims, n, bad_line=None):
    coords = np.stack([rs.integers(1, k + 1, n) for k in dims], 1)
    vals = rs.normal(size=n)
    lines = [" ".join(map(str, c)) + f" {v:.17g}" for c, v in zip(coords, vals)]
    if bad_line is not None:
        lines[bad_line] = lines[bad_line].replace(" ", " z", 1)
    return "#shape: " + " ".join(map(str, dims)) + "\n" + "\n".join(lines) + "\n"


def test_parallel_parse_matches_reference(ref, tmp_path):
    rs = np.random.default_rng(11)
    dims = (300, 200, 100, 50)
    p = tmp_path / "big.tns"
    p.write_text(_big_text(rs, dims, 120_000))  # ~5 MB: the multi-threaded path
    for threads in (1, 3, 16):
        _assert_same_tensor(IO().read_tns(p, threads=threads), ref.read_tns(p))


@pytest.mark.parametrize("bad", [7, 61_234, 119_999])
def test_parallel_parse_reports_first_error_line(ref, tmp_path, bad):
    rs = np.random.default_rng(bad)
    p = tmp_path / "bad.tns"
    p.write_text(_big_text(rs, (50, 60, 70), 120_000, bad_line=bad))
    ours, theirs = _errors(ref, p)
    assert _msg(ours) == _msg(theirs)
    assert f":{bad + 2}:" in _msg(ours)  # header is line 1


@pytest.mark.parametrize("dims", [(30, 40, 50), (3, 2**33, 4)])
def test_binary_coo_roundtrip(tmp_path, dims):
    io = IO()
    rs = np.random.default_rng(1)
    n = 5000
    coords = np.stack([rs.integers(0, k, n) for k in dims], 1)
    t = io.CooTensor(dims, coords, rs.normal(size=n))
    p = tmp_path / "x.coo"
    io.write_coo(t, p)
    width = 4 if max(dims) <= 2**32 else 8
    assert p.stat().st_size == 40 + 8 * len(dims) + n * (width * len(dims) + 8)
    back = io.read_coo(p, threads=4)
    assert back.dims == dims
    assert np.array_equal(back.coords, coords) and np.array_equal(back.values, t.values)
    # truncation / trailing garbage / bad magic are runtime errors naming the file
    g = G()
    raw = p.read_bytes()
    for bad in (raw[:-1], raw + b"\0", b"XXXXXXXX" + raw[8:], raw[:10]):
        p.write_bytes(bad)
        with pytest.raises(g.GcpRuntimeError, match="x.coo"):
            io.read_coo(p)


def test_binary_coo_rejects_out_of_range(tmp_path):
    io, g = IO(), G()
    with pytest.raises(g.OutOfRange):
        io.write_coo(io.CooTensor((3, 4), np.array([[0, 4]]), np.array([1.0])), tmp_path / "y")


def test_dense_roundtrip_matches_reference(ref, tmp_path):
    io = IO()
    rs = np.random.default_rng(2)
    dims = (4, 5, 6)
    vals = rs.normal(size=120)
    p = tmp_path / "d.bin"
    io.write_dense(dims, vals, p)
    rt = ref.read_dense(p)
    assert tuple(rt.dims) == dims and np.array_equal(rt.dense_values(), vals)
    q = tmp_path / "e.bin"
    rt.write_dense(q)
    assert q.read_bytes() == p.read_bytes()
    assert (tmp_path / "e.bin.shape").read_text() == (tmp_path / "d.bin.shape").read_text()
    d2, v2 = io.read_dense(q)
    assert d2 == dims and np.array_equal(v2, vals)
    # short / long files: the reference's messages
    g = G()
    for data in (q.read_bytes()[:-8], q.read_bytes() + b"\0"):
        q.write_bytes(data)
        with pytest.raises(g.GcpRuntimeError) as ours:
            io.read_dense(q)
        with pytest.raises(O.RefError) as theirs:
            ref.read_dense(q)
        assert _msg(ours.value) == _msg(theirs.value)


# ---- model text files and the trace CSV (io.cpp:153-193, 252-260) ----------
def test_model_files_match_reference(ref, tmp_path):
    io = IO()
    rs = np.random.default_rng(4)
    F = [rs.normal(size=(n, 3)) * 10.0 ** rs.integers(-30, 30, (n, 3)) for n in (5, 4, 6)]
    p, q = tmp_path / "ours.model", tmp_path / "ref.model"
    io.write_model(F, p)
    ref.write_model(F, q)
    assert p.read_bytes() == q.read_bytes()
    for got, want in zip(io.read_model(q), F):
        assert np.array_equal(got, want)  # %.17g round trip is bit-exact
    for got, want in zip(ref.read_model(p), F):
        assert np.array_equal(got, want)


@pytest.mark.parametrize("name,text", [
    ("no_header", ""),
    ("bad_header", "3 x\n"),
    ("zero_rank", "2 0\n3 4\n"),
    ("missing_dims", "2 1\n3\n"),
    ("truncated", "2 1\n2 2\n1.0 2.0 3.0\n"),
    ("bad_number", "1 2\n2\n1.0 2.0\n3.0 nope\n"),
])
def test_model_read_errors_match_reference(ref, tmp_path, name, text):
    p = tmp_path / f"{name}.model"
    p.write_text(text)
    g = G()
    with pytest.raises(g.GcpError) as ours:
        IO().read_model(p)
    with pytest.raises(O.RefError) as theirs:
        ref.read_model(p)
    assert _msg(ours.value) == _msg(theirs.value)


def test_trace_csv_matches_reference(ref, tmp_path):
    from paper_1906_01687_b200.fit import FitTraceRecord
    rs = np.random.default_rng(5)
    recs = [FitTraceRecord(i, float(rs.normal() * 1e5), 0.01 * 0.1 ** (i // 3),
                           float(rs.random()), bool(i % 4)) for i in range(12)]
    p, q = tmp_path / "ours.csv", tmp_path / "ref.csv"
    IO().write_trace_csv(recs, p)
    ref.write_trace(q, [t.epoch for t in recs], [t.loss_estimate for t in recs],
                    [t.learning_rate for t in recs], [t.seconds for t in recs],
                    [t.accepted for t in recs])
    assert p.read_bytes() == q.read_bytes()
