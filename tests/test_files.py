"""Matrix Market ingestion / output and the SKRYRCY1 recycle-space dump
(SURVEY.md §8 row f3), host side of the C-ABI — the cases of the reference's
proj/tests/test_matrix_market.cpp and test_recycle.cpp:252-290. CPU only."""
import os

import numpy as np
import pytest
import scipy.sparse as sp


@pytest.fixture(scope="module")
def sk():
    import paper_2311_14206_b200 as sk
    return sk


def dense(csr):
    rows, cols, off, col, val = csr
    return sp.csr_matrix((val, col, off), shape=(rows, cols)).toarray()


def test_coordinate_general_round_trips_bit_exactly(sk):
    rng = np.random.default_rng(21)
    r, c = rng.integers(0, 9, 40), rng.integers(0, 9, 40)
    v = rng.standard_normal(40) * 10.0 ** (np.arange(40) % 7 - 3.0)
    A = sp.coo_matrix((v, (r, c)), shape=(9, 9)).tocsr()
    A.sum_duplicates()
    A.eliminate_zeros()
    text = sk.matrix_market_string(9, 9, A.indptr, A.indices, A.data)
    assert text.startswith("%%MatrixMarket matrix coordinate real general\n9 9 ")
    B = sk.read_matrix_market(text=text)
    assert np.array_equal(dense(B), A.toarray())  # 17 significant digits round-trip exactly
    assert np.array_equal(B[2], A.indptr) and np.array_equal(B[3], A.indices) and np.array_equal(B[4], A.data)


def test_symmetric_coordinate_entries_are_mirrored(sk):
    B = sk.read_matrix_market(text="%%MatrixMarket matrix coordinate real symmetric\n3 3 4\n"
                                   "1 1 2.0\n2 1 -1.0\n3 2 0.5\n3 3 4.0\n")
    assert np.array_equal(dense(B), [[2.0, -1.0, 0.0], [-1.0, 0.0, 0.5], [0.0, 0.5, 4.0]])


def test_integer_values_and_array_format(sk):
    B = sk.read_matrix_market(text="%%MatrixMarket matrix coordinate integer general\n% a comment line\n"
                                   "2 2 2\n1 1 3\n2 2 -7\n")
    assert dense(B)[0, 0] == 3.0 and dense(B)[1, 1] == -7.0
    C = sk.read_matrix_market(text="%%MatrixMarket matrix array real general\n2 3\n1\n2\n3\n4\n5\n6\n")
    assert np.array_equal(dense(C), [[1, 3, 5], [2, 4, 6]])  # column-major order


def test_array_symmetric_reads_lower_triangle(sk):
    B = sk.read_matrix_market(text="%%MatrixMarket matrix array real symmetric\n3 3\n1\n2\n3\n4\n5\n6\n")
    assert np.array_equal(dense(B), [[1, 2, 3], [2, 4, 5], [3, 5, 6]])


@pytest.mark.parametrize("text", [
    "%%MatrixMarket matrix coordinate complex general\n1 1 1\n1 1 1 0\n",
    "%%MatrixMarket matrix coordinate pattern general\n1 1 1\n1 1\n",
    "%%MatrixMarket matrix coordinate real skew-symmetric\n1 1 0\n",
    "not a header\n",
])
def test_unsupported_headers_rejected(sk, text):
    with pytest.raises(RuntimeError):
        sk.read_matrix_market(text=text)


def test_parse_errors_carry_line_number(sk):
    with pytest.raises(RuntimeError, match="line 3"):
        sk.read_matrix_market(text="%%MatrixMarket matrix coordinate real general\n2 2 1\n5 1 1.0\n")
    with pytest.raises(RuntimeError, match="unexpected end of data"):
        sk.read_matrix_market(text="%%MatrixMarket matrix coordinate real general\n2 2 1\n")
    with pytest.raises(RuntimeError, match="line 4"):
        sk.read_matrix_market(text="%%MatrixMarket matrix coordinate real general\n2 2 2\n1 1 1.0\n2 2 zz\n")


def test_duplicates_summed_and_zeros_dropped(sk):
    B = sk.read_matrix_market(text="%%MatrixMarket matrix coordinate real general\n2 2 5\n"
                                   "1 1 1.5\n1 1 2.5\n2 1 1.0\n2 2 1.0\n2 2 -1.0\n")
    assert dense(B)[0, 0] == 4.0 and dense(B)[1, 0] == 1.0
    assert len(B[4]) == 2  # (2,2) summed to an exact zero and dropped (sparse.hpp:65)


def test_file_wrappers_round_trip_and_missing_file(sk, tmp_path):
    path = str(tmp_path / "mm_roundtrip_test.mtx")
    sk.write_matrix_market(path, 2, 2, [0, 1, 2], [1, 0], [3.25, -1.0])
    B = sk.read_matrix_market(path)
    assert np.array_equal(dense(B), [[0.0, 3.25], [-1.0, 0.0]])
    with pytest.raises(RuntimeError, match="cannot open Matrix Market file"):
        sk.read_matrix_market("definitely_missing_file.mtx")


def _space(seed, n=10, s=6, k=4):
    rng = np.random.default_rng(seed)
    return (np.asfortranarray(rng.standard_normal((n, k))), np.asfortranarray(rng.standard_normal((s, k))),
            np.asfortranarray(rng.standard_normal((s, k))))


def test_space_file_round_trip_and_layout(sk, tmp_path):
    U, SU, SAU = _space(70)
    data = sk.space_file_bytes(U, SU, SAU, provenance="exact-resketch")
    # magic, n, s, k, provenance (native int64), then U, SU, SAU column-major
    assert data[:8] == b"SKRYRCY1"
    assert np.array_equal(np.frombuffer(data[8:40], dtype=np.int64), [10, 6, 4, 3])
    assert np.array_equal(np.frombuffer(data[40:40 + 8 * 40]), U.ravel(order="F"))
    back = sk.read_space_file(data=data)
    assert back["provenance"] == "exact-resketch" and (back["n"], back["s"], back["k"]) == (10, 6, 4)
    assert np.array_equal(back["U"], U) and np.array_equal(back["SU"], SU) and np.array_equal(back["SAU"], SAU)
    path = str(tmp_path / "space.bin")
    with open(path, "wb") as fh:
        fh.write(data)
    again = sk.read_space_file(path)
    assert np.array_equal(again["SAU"], SAU)


def test_space_file_rejects_bad_input(sk):
    U, SU, SAU = _space(71)
    with pytest.raises(RuntimeError, match="bad magic"):
        sk.read_space_file(data=b"NOTASPACEFILE\x01\x02\x03\x04\x05\x06\x07\x08")
    full = sk.space_file_bytes(U, SU, SAU)
    with pytest.raises(RuntimeError, match="truncated"):
        sk.read_space_file(data=full[:len(full) // 2])
    bad = bytearray(full)
    bad[32:40] = np.array([9], dtype=np.int64).tobytes()  # provenance out of range
    with pytest.raises(RuntimeError, match="corrupt header"):
        sk.read_space_file(data=bytes(bad))
    with pytest.raises(RuntimeError, match="cannot open recycle-space file"):
        sk.read_space_file("/nonexistent/path/space.bin")


def test_matrix_market_random_round_trips(sk):
    """Randomised round trips (shapes incl. empty rows / columns, 1 x n,
    values over many magnitudes): write -> read reproduces the CSR exactly,
    and the symmetric form mirrors the lower triangle."""
    rng = np.random.default_rng(123)
    for trial in range(25):
        rows, cols = int(rng.integers(1, 40)), int(rng.integers(1, 40))
        nnz = int(rng.integers(0, rows * cols + 1))
        r = rng.integers(0, rows, nnz)
        c = rng.integers(0, cols, nnz)
        v = rng.standard_normal(nnz) * 10.0 ** rng.integers(-12, 12, nnz)
        A = sp.coo_matrix((v, (r, c)), shape=(rows, cols)).tocsr()
        A.sum_duplicates()
        A.eliminate_zeros()
        text = sk.matrix_market_string(rows, cols, A.indptr, A.indices, A.data)
        B = sk.read_matrix_market(text=text)
        assert B[0] == rows and B[1] == cols
        assert np.array_equal(B[2], A.indptr) and np.array_equal(B[3], A.indices)
        assert np.array_equal(B[4], A.data)
    # symmetric coordinate: the mirror of a random lower triangle
    n = 25
    L = sp.tril(sp.random(n, n, density=0.2, random_state=5)).tocoo()
    body = "".join(f"{i + 1} {j + 1} {float(x)!r}\n" for i, j, x in zip(L.row, L.col, L.data))
    S = sk.read_matrix_market(text=f"%%MatrixMarket matrix coordinate real symmetric\n{n} {n} {L.nnz}\n{body}")
    D = L.toarray()
    ref = D + D.T - np.diag(np.diag(D))
    got = sp.csr_matrix((S[4], S[3], S[2]), shape=(n, n)).toarray()
    assert np.array_equal(got, ref)
