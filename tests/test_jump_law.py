"""The lattice-jump law (walk.cu `jump_law`, host-only C ABI
frw_lattice_jump_law) against an independent sparse solve of the simple
symmetric walk's Green's function on the (2m-1)^3 interior of the L-inf
sphere of radius m: P(first hit = b) = G(x_b, c) / 6 over b's interior
neighbour x_b, E[tau] = sum_x G(x, c).  Also checked: the face law is
symmetric under the square's dihedral group, and a plain Monte Carlo of the
walk (numpy) agrees with it."""
import numpy as np
import pytest
import scipy.sparse as sp
import scipy.sparse.linalg as spl

from paper_2507_09730_b200 import capi


def _srw_green(m):
    s = 2 * m - 1
    idx = np.arange(s ** 3).reshape(s, s, s)
    rows, cols = [], []
    for ax in range(3):
        a = np.moveaxis(idx, ax, 0)
        rows += [a[:-1].ravel(), a[1:].ravel()]
        cols += [a[1:].ravel(), a[:-1].ravel()]
    r, c = np.concatenate(rows), np.concatenate(cols)
    P = sp.csr_matrix((np.full(len(r), 1 / 6), (r, c)), shape=(s ** 3, s ** 3))
    A = sp.identity(s ** 3, format="csr") - P
    b = np.zeros(s ** 3)
    b[idx[m - 1, m - 1, m - 1]] = 1.0
    G = spl.spsolve(A.tocsc(), b)  # A symmetric: G(x, c) = G(c, x)
    return G.reshape(s, s, s)


@pytest.mark.parametrize("m", [2, 3, 5, 8, 11])
def test_jump_law_matches_sparse_solve(m):
    face, et = capi.lattice_jump_law(m)
    G = _srw_green(m)
    # face -x: hit (0 - 1, j, k) from interior node (0, j, k); array is
    # [v][u] = [z][y]
    want = G[0, :, :].T / 6.0
    assert np.allclose(face, want, rtol=1e-10, atol=1e-15)
    assert abs(6 * face.sum() - 1.0) < 1e-12
    assert abs(et - G.sum()) < 1e-9 * G.sum()
    # dihedral symmetry of the face
    assert np.allclose(face, face.T, atol=1e-15)
    assert np.allclose(face, face[::-1, :], atol=1e-15)


def test_jump_law_m2_closed_form_and_monte_carlo():
    face, et = capi.lattice_jump_law(2)
    # E[tau] for radius 2: from the centre one step to a face node of the
    # 3^3 interior, then the walk on the 27 interior nodes
    G = _srw_green(2)
    assert abs(et - G.sum()) < 1e-12
    rng = np.random.default_rng(3)
    W = 200_000
    p = np.zeros((W, 3), np.int64)
    steps = np.zeros(W, np.int64)
    alive = np.ones(W, bool)
    moves = np.array([[-1, 0, 0], [1, 0, 0], [0, -1, 0], [0, 1, 0], [0, 0, -1], [0, 0, 1]])
    while alive.any():
        k = np.flatnonzero(alive)
        p[k] += moves[rng.integers(0, 6, len(k))]
        steps[k] += 1
        alive[k] = np.abs(p[k]).max(axis=1) < 2
    on = p[:, 0] == -2
    h = np.zeros((3, 3))
    np.add.at(h, (p[on, 2] + 1, p[on, 1] + 1), 1)
    assert abs(on.mean() - 1 / 6) < 4 * np.sqrt(1 / 6 * 5 / 6 / W)
    assert np.allclose(h / W, face, atol=4 * np.sqrt(face.max() / W))
    assert abs(steps.mean() - et) < 4 * steps.std() / np.sqrt(W)


def test_jump_law_rejects_bad_radius():
    with pytest.raises(capi.FrwError):
        capi.lattice_jump_law(1)
    with pytest.raises(capi.FrwError):
        capi.lattice_jump_law(32)
