# SPDX-License-Identifier: Apache-2.0
"""MatrixMarket ingestion: the native loader/writer in
libpcgx.so against the reference's load_matrix_market / save_matrix_market
(matrix_market.cpp:55-199). Every case of tests/golden/mm_cases.py must give the
reference's CSR arrays bitwise (SHA-256 of the int64 / float64 bytes) or the
reference's ParseError message verbatim; saved text must be byte-identical.
Host-only (no GPU); when oracle/_ref is built the reference runs live too."""
import hashlib
import os

import numpy as np
import pytest

from tests._util import sha
from tests.golden.mm_cases import cases

CASES = cases()


def _sha_i64(a):
    return hashlib.sha256(np.ascontiguousarray(a, dtype="<i8").tobytes()).hexdigest()


@pytest.fixture(scope="module")
def ref():
    from oracle.oracle import RefLib
    try:
        return RefLib()
    except FileNotFoundError:
        return None


@pytest.mark.parametrize("name", sorted(CASES))
def test_load_matches_reference_golden(pcgx, golden, name):
    g = golden["matrix_market"][name]
    text = CASES[name]
    if "error" in g:
        with pytest.raises(pcgx.ParseError) as ei:
            pcgx.load_matrix_market(text, name="<" + name + ">")
        assert str(ei.value) == g["error"]
        return
    m = pcgx.load_matrix_market(text, name="<" + name + ">")
    assert (m.n, len(m.values)) == (g["n"], g["nnz"])
    assert _sha_i64(m.row_ptr) == g["row_ptr"]
    assert _sha_i64(m.col_idx) == g["col_idx"]
    assert sha(m.values) == g["values"]
    saved = pcgx.save_matrix_market(m)
    assert hashlib.sha256(saved.encode()).hexdigest() == g["save_sha256"]
    back = pcgx.load_matrix_market(saved, name="<roundtrip>")  # load(save(m)) == m
    assert np.array_equal(back.row_ptr, m.row_ptr) and np.array_equal(back.col_idx, m.col_idx)
    assert np.array_equal(back.values.view(np.uint64), m.values.view(np.uint64))


@pytest.mark.parametrize("name", ["lap2d160_sym_big", "lap2d30_general_shuffled", "crlf",
                                  "lap2d160_sym_big_error", "num_hexfloat", "dup_general"])
def test_load_matches_reference_live(pcgx, ref, name):
    if ref is None:
        pytest.skip("oracle/_ref not built (no /root/reference here)")
    from oracle.oracle import OracleError
    text = CASES[name]
    try:
        n, rp, ci, va = ref.mm_load(text, "<x>")
    except OracleError as e:
        with pytest.raises(pcgx.ParseError) as ei:
            pcgx.load_matrix_market(text, name="<x>")
        assert str(ei.value) == str(e)
        return
    m = pcgx.load_matrix_market(text, name="<x>")
    assert m.n == n and np.array_equal(m.row_ptr, rp) and np.array_equal(m.col_idx, ci)
    assert np.array_equal(m.values.view(np.uint64), va.view(np.uint64))
    assert pcgx.save_matrix_market(m) == ref.mm_save(n, rp, ci, va)


def test_file_path_variants(pcgx, tmp_path, golden):
    # test_matrix_market.cpp:121-129
    A = pcgx.gen_fe27(6, sigma=1.0, seed=20240801)
    m = pcgx.CsrMatrix(A.n, A.row_ptr.astype(np.int64), A.col_idx.astype(np.int64), A.values)
    path = tmp_path / "fe27_6.mtx"
    pcgx.save_matrix_market(m, str(path))
    text = path.read_text()
    assert text.splitlines()[0] == "%%MatrixMarket matrix coordinate real symmetric"
    assert text == pcgx.save_matrix_market(m)
    back = pcgx.load_matrix_market(str(path))
    assert np.array_equal(back.row_ptr, m.row_ptr) and np.array_equal(back.col_idx, m.col_idx)
    assert np.array_equal(back.values, m.values)
    with pytest.raises(pcgx.ParseError) as ei:
        pcgx.load_matrix_market("does_not_exist.mtx")
    assert str(ei.value) == "does_not_exist.mtx: cannot open file"
    # a path's errors are reported with the path as the name
    bad = tmp_path / "bad.mtx"
    bad.write_bytes(CASES["zero_based"])
    with pytest.raises(pcgx.ParseError) as ei:
        pcgx.load_matrix_market(str(bad))
    assert str(ei.value) == f"{bad}:3: index (0, 0) out of range for 1-based indices in [1, 2]"


def test_roundtrip_non_representable_values(pcgx):
    # test_matrix_market.cpp:103-119: 17 significant digits survive save/load
    vals = pcgx.random_uniform_vector(8, 4242)
    rows, cols, v = [], [], []
    for i in range(8):
        rows.append(i), cols.append(i), v.append(3.0 + vals[i] / 3.0)
    t = sorted(zip(rows + [5, 2], cols + [2, 5], v + [vals[0] / 7.0, vals[0] / 7.0]))
    rp = np.zeros(9, dtype=np.int64)
    for r, _, _ in t:
        rp[r + 1] += 1
    rp = np.cumsum(rp)
    m = pcgx.CsrMatrix(8, rp, np.array([c for _, c, _ in t], dtype=np.int64),
                       np.array([x for _, _, x in t]))
    back = pcgx.load_matrix_market(pcgx.save_matrix_market(m), name="<roundtrip>")
    assert np.array_equal(back.row_ptr, m.row_ptr) and np.array_equal(back.col_idx, m.col_idx)
    assert np.array_equal(back.values.view(np.uint64), m.values.view(np.uint64))
