"""CPU tests: pin the oracle (test infrastructure) before trusting it.

1. The C restatement (oracle/rvk_oracle.c) is bit-identical to the
   reference's own kernels compiled from /root/reference/proj/src
   (oracle/_ref) on every kernel and on whole CG solves.
2. It reproduces the committed golden vectors (tests/golden/cg_golden.json,
   generated from oracle/_ref by tests/golden/make_golden.py).
3. It satisfies the SPEC.md known answers (:363-409, :464, :483-484,
   :532-547) and the stencil closed forms.
"""
import hashlib
import json
import os

import numpy as np
import pytest

import oracle as O

GOLDEN = os.path.join(os.path.dirname(__file__), "golden", "cg_golden.json")


def _sha(a):
    return hashlib.sha256(np.ascontiguousarray(a).tobytes()).hexdigest()


def _fromhex(lst):
    return np.array([float.fromhex(v) for v in lst])


@pytest.fixture(scope="module")
def golden():
    with open(GOLDEN) as f:
        return json.load(f)


needs_ref = pytest.mark.skipif(not O.ref_available(), reason="oracle/_ref not built")


# ---- golden vectors ------------------------------------------------------------
def test_golden_cases_cover_spec_grids(golden):
    names = {c["name"] for c in golden["cases"]}
    for want in ("5pt_16x16", "5pt_32x32", "9pt_16x16", "9pt_32x32", "7pt_8x8x8", "27pt_8x8x8"):
        assert want in names


def test_oracle_matches_golden_bitwise(golden):
    for c in golden["cases"]:
        A = O.build_laplacian(c["dim"], c["points"], c["grid"])
        assert A.n_rows == c["n"] and A.nnz == c["nnz"], c["name"]
        assert _sha(A.off) == c["sha_off"], c["name"]
        assert _sha(A.cols) == c["sha_cols"], c["name"]
        assert _sha(A.vals) == c["sha_vals"], c["name"]
        b = O.rhs(A.n_rows)
        assert _sha(b) == c["sha_b"], c["name"]
        assert np.array_equal(O.spmv(A, b), _fromhex(c["spmv_b"])), c["name"]
        r = O.cg_solve(A, b, max_it=golden["max_it"], pc=c["pc"])
        assert r.status == c["status"] and r.iterations == c["iterations"], c["name"]
        assert np.array_equal(r.hist, _fromhex(c["hist"])), c["name"]
        assert np.array_equal(r.x, _fromhex(c["x"])), c["name"]


# ---- restatement vs the reference's own kernels ------------------------------
@needs_ref
@pytest.mark.parametrize("n", [0, 1, 3, 4, 7, 1000, 4099])
def test_vec_kernels_match_reference(n):
    rng = np.random.default_rng(n + 1)
    x, y = rng.standard_normal(n), rng.standard_normal(n)
    R, L = O.ref_lib(), O.lib()
    assert R.ref_dot(0, n, x, y) == L.ro_dot(n, x, y)
    assert R.ref_nrm2(0, n, x) == L.ro_nrm2(n, x)
    for name in ("axpy", "aypx"):
        y1, y2 = y.copy(), y.copy()
        getattr(R, "ref_" + name)(0, n, 0.37, x, y1)
        getattr(L, "ro_" + name)(n, 0.37, x, y2)
        assert np.array_equal(y1, y2), name
        # elementwise kernels are bit-identical across reference backends (kernels.hpp:7-10)
        if O.ref_lib().ref_avx2_supported():
            y3 = y.copy()
            getattr(R, "ref_" + name)(1, n, 0.37, x, y3)
            assert np.array_equal(y1, y3), name
    w1, w2 = np.empty(n), np.empty(n)
    R.ref_waxpy(n, -1.25, x, y, w1)
    L.ro_waxpy(n, -1.25, x, y, w2)
    assert np.array_equal(w1, w2)
    s1, s2 = x.copy(), x.copy()
    R.ref_scale(n, 3.5, s1)
    L.ro_scale(n, 3.5, s2)
    assert np.array_equal(s1, s2)
    p1, p2 = np.empty(n), np.empty(n)
    R.ref_pointwise_mult(0, n, x, y, p1)
    L.ro_pointwise_mult(n, x, y, p2)
    assert np.array_equal(p1, p2)


@needs_ref
@pytest.mark.parametrize("spec", [(2, 5, (33, 17)), (2, 9, (20, 21)), (3, 7, (9, 8, 7)),
                                  (3, 27, (7, 6, 5))])
def test_spmv_matches_reference_scalar(spec):
    A = O.build_laplacian(*spec)
    x = np.random.default_rng(0).standard_normal(A.n_rows)
    assert np.array_equal(O.spmv(A, x), O.ref_spmv(A, x, backend=0))


@needs_ref
@pytest.mark.parametrize("spec", [(2, 5, (64, 64)), (2, 9, (48, 40)), (3, 7, (16, 16, 16)),
                                  (3, 27, (12, 12, 12))])
def test_cg_restatement_matches_reference_kernels(spec):
    A = O.build_laplacian(*spec)
    b = O.rhs(A.n_rows)
    r1 = O.cg_solve(A, b)
    r2 = O.ref_cg_solve(A, b, backend=0)
    assert np.array_equal(r1.hist, r2.hist) and np.array_equal(r1.x, r2.x)
    # the AVX2 backend reorders the reductions: within 1e-10
    if O.ref_lib().ref_avx2_supported():
        r3 = O.ref_cg_solve(A, b, backend=1)
        assert np.max(np.abs(r3.hist - r1.hist) / r1.hist) < 1e-12


# ---- SPEC known answers -----------------------------------------------------------
def test_spec_stencil_known_answers():
    A = O.build_laplacian(2, 5, (3, 3))
    centre = A.off[4], A.off[5]
    assert list(A.vals[centre[0]:centre[1]]) == [-1, -1, 4, -1, -1]
    assert A.off[1] - A.off[0] == 3  # corner row has 3 entries
    A = O.build_laplacian(3, 7, (2, 2, 2))  # 4 entries per row
    assert np.all(np.diff(A.off) == 4)
    for dim, pts, centre_v in [(2, 5, 4), (3, 7, 6), (2, 9, 8), (3, 27, 26)]:
        g = (5, 5) if dim == 2 else (4, 4, 4)
        A = O.build_laplacian(dim, pts, g)
        d = O.diagonal(A)
        assert np.all(d == centre_v)
        assert set(np.unique(A.vals)) == {-1.0, float(centre_v)}


@pytest.mark.parametrize("N", [2, 3, 5, 8, 13])
def test_stencil_nnz_closed_forms(N):
    # brute force (the builder) vs the closed forms of SURVEY.md 8c
    assert O.build_laplacian(2, 5, (N, N)).nnz == 5 * N * N - 4 * N
    assert O.build_laplacian(2, 9, (N, N)).nnz == (3 * N - 2) ** 2
    assert O.build_laplacian(3, 7, (N, N, N)).nnz == 7 * N ** 3 - 6 * N * N
    assert O.build_laplacian(3, 27, (N, N, N)).nnz == (3 * N - 2) ** 3


@pytest.mark.parametrize("spec", [(2, 5, (8, 8)), (2, 9, (8, 8)), (3, 7, (4, 4, 4)),
                                  (3, 27, (4, 4, 4))])
def test_stencil_symmetric_spd(spec):
    # symmetric (exact) and SPD (dense eigensolve, <= 8/dim)
    A = O.build_laplacian(*spec)
    D = np.zeros((A.n_rows, A.n_rows))
    for r in range(A.n_rows):
        for k in range(A.off[r], A.off[r + 1]):
            D[r, A.cols[k]] = A.vals[k]
    assert np.array_equal(D, D.T)
    assert np.linalg.eigvalsh(D).min() > 0
    # columns strictly increasing within each row (csr.hpp:51-53)
    for r in range(A.n_rows):
        assert np.all(np.diff(A.cols[A.off[r]:A.off[r + 1]]) > 0)


def test_invalid_stencil_rejected():
    for spec in [(2, 7, (4, 4)), (3, 5, (4, 4, 4)), (2, 5, (1, 4)), (4, 5, (2, 2))]:
        with pytest.raises(ValueError):
            O.build_laplacian(*spec)


def test_spec_vec_and_spmv_known_answers():
    L = O.lib()
    assert O.nrm2([3.0, 4.0]) == 5.0
    assert O.nrm2(np.zeros(100)) == 0.0                    # :364
    assert O.dot([1.0, 1, 1], [1.0, 1, 1]) == 3.0          # :381
    assert O.dot([1.0, 0], [0.0, 1]) == 0.0                # :382
    y = np.array([1.0, 1.0])
    L.ro_axpy(2, 2.0, np.array([3.0, 4.0]), y)            # :391
    assert list(y) == [7.0, 9.0]
    v = np.array([3.0, 4.0])
    L.ro_scale(2, 1.0 / O.nrm2(v), v)                      # :372 normalize
    assert np.allclose(v, [0.6, 0.8], rtol=0, atol=1e-15)
    # 1D 3-point Laplacian [2,-1;-1,2,-1;-1,2] * 1 = [1,0,1]  (:409)
    A = O.Csr(3, 3, np.array([0, 2, 5, 7], np.int64), np.array([0, 1, 0, 1, 2, 1, 2], np.int32),
              np.array([2.0, -1, -1, 2, -1, -1, 2]))
    assert list(O.spmv(A, np.ones(3))) == [1.0, 0.0, 1.0]
    # identity -> y = x (:408)
    I = O.Csr(4, 4, np.arange(5, dtype=np.int64), np.arange(4, dtype=np.int32), np.ones(4))
    x = np.array([1.5, -2.0, 3.25, 0.0])
    assert np.array_equal(O.spmv(I, x), x)
    # Jacobi: diag [2,4], r [2,4] -> z [1,1] (:483)
    z = np.empty(2)
    L.ro_pointwise_mult(2, 1.0 / np.array([2.0, 4.0]), np.array([2.0, 4.0]), z)
    assert list(z) == [1.0, 1.0]


def test_cg_identity_converges_in_one_iteration():
    # A = I, pc = None -> converges in 1 iteration, x = b
    n = 50
    I = O.Csr(n, n, np.arange(n + 1, dtype=np.int64), np.arange(n, dtype=np.int32), np.ones(n))
    b = O.rhs(n)
    r = O.cg_solve(I, b, pc="none")
    assert r.status == 1 and r.iterations == 1
    assert np.array_equal(r.x, b)


def test_cg_breakdown_reported_with_iteration():
    # indefinite A = diag(1, -1), b = [1, 1]: p.Ap = 0 at iteration 0
    A = O.Csr(2, 2, np.array([0, 1, 2], np.int64), np.array([0, 1], np.int32),
              np.array([1.0, -1.0]))
    r = O.cg_solve(A, np.array([1.0, 1.0]), pc="none")
    assert r.status == 2 and r.breakdown_iter == 0


def test_cg_rtol_early_exit():
    A = O.build_laplacian(2, 5, (16, 16))
    b = O.rhs(A.n_rows)
    full = O.cg_solve(A, b, max_it=200)
    r = O.cg_solve(A, b, max_it=200, rtol=1e-6)
    assert r.status == 1
    k = r.iterations
    assert r.hist[k] <= 1e-6 * r.hist[0] < r.hist[k - 1]
    assert np.array_equal(r.hist, full.hist[: k + 1])


def test_rhs_in_range_and_exact():
    b = O.rhs(10000)
    assert b.min() >= -1.0 and b.max() < 1.0
    # exactly k * 2^-52 - 1 for an integer k < 2^53
    k = (b + 1.0) * 2.0 ** 52
    assert np.array_equal(k, np.round(k))


# ---- the large-size restatement (oracle/rvk_oracle_mt.c) ------------------------
LARGE_SPECS = [(2, 5, (37, 29)), (2, 9, (64, 41)), (3, 7, (17, 13, 11)), (3, 27, (12, 10, 9)),
               (2, 5, (2, 2)), (3, 27, (2, 3, 2))]


@pytest.mark.parametrize("spec", LARGE_SPECS)
def test_build_laplacian_rows_is_a_slice_of_the_full_build(spec):
    """Row slabs (the 768^3 device-assembly check) equal the full build's
    rows bit for bit; the running nnz reproduces the global offsets."""
    dim, pts, g = spec
    A = O.build_laplacian(dim, pts, g)
    rng = np.random.default_rng(len(g) * 100 + pts)
    cuts = np.unique(np.concatenate([[0, A.n_rows], rng.integers(0, A.n_rows, 5)]))
    base = 0
    for r0, r1 in zip(cuts[:-1], cuts[1:]):
        off, cols, vals = O.build_laplacian_rows(dim, pts, g, int(r0), int(r1))
        assert np.array_equal(off + base, A.off[r0:r1 + 1])
        assert np.array_equal(cols, A.cols[A.off[r0]:A.off[r1]])
        assert np.array_equal(vals.view(np.uint64), A.vals[A.off[r0]:A.off[r1]].view(np.uint64))
        base += int(off[-1])
    assert base == A.nnz


@pytest.mark.parametrize("spec", LARGE_SPECS)
def test_stencil_spmv_bitexact_vs_csr(spec):
    dim, pts, g = spec
    A = O.build_laplacian(dim, pts, g)
    x = np.random.default_rng(7).standard_normal(A.n_rows)
    assert np.array_equal(O.stencil_spmv(dim, pts, g, x).view(np.uint64), O.spmv(A, x).view(np.uint64))


@pytest.mark.parametrize("spec", LARGE_SPECS[:4] + [(3, 7, (64, 64, 40)), (2, 9, (400, 300))])
@pytest.mark.parametrize("pc", ["jacobi", "none"])
def test_threaded_stencil_cg_matches_serial_oracle(spec, pc):
    """The threaded matrix-free PCG (used at 768^3) is the serial oracle's
    loop with chunked reductions: history and x within 1e-13."""
    dim, pts, g = spec
    A = O.build_laplacian(dim, pts, g)
    b = O.rhs(A.n_rows)
    ref = O.cg_solve(A, b, max_it=20, pc=pc)
    got = O.cg_solve_stencil(dim, pts, g, b, max_it=20, pc=pc)
    assert got.iterations == ref.iterations and got.status == ref.status
    keep = ref.hist > 1e-8 * ref.hist[0]
    assert np.max(np.abs(got.hist[keep] - ref.hist[keep]) / ref.hist[keep]) < 1e-13
    assert np.linalg.norm(got.x - ref.x) <= 1e-13 * np.linalg.norm(ref.x)
