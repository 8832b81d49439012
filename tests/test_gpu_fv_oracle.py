"""The full-domain finite-volume reference (reference_capacitance,
oracle.cpp:92-213) on the device: pinned against a scipy restatement of the
same discretisation at small resolution, Maxwell-consistent, and used as the
reference's end-to-end acceptance pin (acceptance_main.cpp:380-413: FRW
HYBRID-MW N=24 within 5% err_avg of the R=144 solution on the four
fixtures)."""
import json

import numpy as np
import pytest
import scipy.sparse as sp
import scipy.sparse.linalg as spla

import paper_2507_09730_b200.frwcap as frwcap
from tests import scenes

pytestmark = pytest.mark.gpu
EPS0 = 8.8541878128e-12


def _scipy_fv(sc, R):
    """numpy/scipy restatement of oracle.cpp:92-213 (direct solve)"""
    lo, hi = sc.world[:3], sc.world[3:]
    h = (hi - lo) / R
    fpre = np.array([h[1] * h[2] / h[0], h[0] * h[2] / h[1], h[0] * h[1] / h[2]])
    idx = np.arange(R ** 3)
    i, j, k = idx % R, (idx // R) % R, idx // (R * R)
    p = np.stack([lo[0] + (i + 0.5) * h[0], lo[1] + (j + 0.5) * h[1], lo[2] + (k + 0.5) * h[2]], 1)
    eps = np.full(R ** 3, float(sc.background_eps))
    for b, e in zip(sc.diel_box.reshape(-1, 6), sc.diel_eps):
        inside = np.all((p >= b[:3]) & (p <= b[3:]), axis=1)
        eps[inside] = e
    term = np.full(R ** 3, -1)
    for t in range(sc.n_cond - 1, -1, -1):
        b = sc.cond_box[t]
        inside = np.all((p >= b[:3]) & (p <= b[3:]), axis=1)
        term[inside] = t
    free = term < 0
    row = -np.ones(R ** 3, int)
    row[free] = np.arange(free.sum())
    rows, cols, vals = [], [], []
    diag = np.zeros(free.sum())
    faces = []  # (row, term, g)
    coords = [i, j, k]
    for d in range(6):
        a = d >> 1
        sgn = 1 if d & 1 else -1
        nc = coords[a] + sgn
        st = [1, R, R * R][a]
        v = idx[free]
        ncv = nc[free]
        ev = eps[free]
        wall = (ncv < 0) | (ncv >= R)
        g_wall = 2.0 * fpre[a] * ev
        diag += np.where(wall, g_wall, 0.0)
        u = np.where(wall, 0, v + sgn * st)
        tu = np.where(wall, -1, term[u])
        cond = (~wall) & (tu >= 0)
        diag += np.where(cond, g_wall, 0.0)
        for rr, tt, gg in zip(row[v][cond], tu[cond], g_wall[cond]):
            faces.append((rr, tt, gg))
        fr = (~wall) & (tu < 0)
        en = eps[u]
        g = fpre[a] * 2.0 * ev * en / (ev + en)
        diag += np.where(fr, g, 0.0)
        rows.append(row[v][fr])
        cols.append(row[u[fr]])
        vals.append(-g[fr])
    n = free.sum()
    A = sp.csr_matrix((np.concatenate(vals + [diag]),
                       (np.concatenate(rows + [np.arange(n)]), np.concatenate(cols + [np.arange(n)]))),
                      shape=(n, n))
    faces = np.array(faces)
    T = sc.n_cond
    cap = np.zeros((T, T))
    lu = spla.splu(A.tocsc())
    for t in range(T):
        b = np.zeros(n)
        sel = faces[:, 1] == t
        np.add.at(b, faces[sel, 0].astype(int), faces[sel, 2])
        phi = lu.solve(b)
        q = np.zeros(T)
        v_term = (faces[:, 1] == t).astype(float)
        np.add.at(q, faces[:, 1].astype(int), faces[:, 2] * (v_term - phi[faces[:, 0].astype(int)]))
        cap[:, t] = q * (EPS0 * 1e-9)
    return cap


def _file(tmp_path, sc, name="s.json"):
    f = tmp_path / name
    f.write_text(sc.to_json())
    return str(f)


@pytest.mark.parametrize("name", ["highk_cross", "conformal_staircase", "stratified_stack"])
def test_fv_matches_scipy_restatement(tmp_path, name):
    sc = scenes.load_fixture(name)
    R = 20
    d = frwcap.reference_capacitance_file(_file(tmp_path, sc), resolution=R)
    cap = np.array(d["capacitance_farads"])
    ref = _scipy_fv(sc, R)
    assert list(d["terminal_ids"]) == [int(x) for x in sc.cond_id]
    assert np.allclose(cap, ref, rtol=1e-6, atol=1e-9 * np.abs(ref).max())
    assert d["residual"] <= 1e-9


def test_fv_maxwell_properties(tmp_path):
    sc = scenes.load_fixture("highk_cross")
    cap = np.array(frwcap.reference_capacitance_file(_file(tmp_path, sc), resolution=48)
                   ["capacitance_farads"])
    assert (np.diag(cap) > 0).all()
    off = cap[~np.eye(len(cap), dtype=bool)]
    assert (off < 0).all()
    # diagonal dominance: with every conductor at 1 V the grounded wall
    # still draws charge, so each row sums to the (positive) ground coupling
    assert (cap.sum(axis=1) >= 0).all()
    assert np.allclose(cap, cap.T, rtol=1e-5)


def test_fv_input_checks(tmp_path):
    sc = scenes.load_fixture("highk_cross")
    with pytest.raises(ValueError):
        frwcap.reference_capacitance_file(_file(tmp_path, sc), resolution=8)
    with pytest.raises(ValueError):
        frwcap.reference_capacitance_file(_file(tmp_path, sc), resolution=200)


@pytest.mark.parametrize("name", list(scenes.FIXTURE_NAMES))
def test_acceptance_frw_within_5pct_of_fv(tmp_path, name):
    """acceptance_main.cpp:339-413: err_avg <= 0.05 at R = 144"""
    sc = scenes.load_fixture(name)
    path = _file(tmp_path, sc)
    ref = frwcap.reference_capacitance_file(path, resolution=144)
    cap = np.array(ref["capacitance_farads"])
    ids = list(ref["terminal_ids"])
    res = frwcap.extract_file(path, mode="HYBRID-MW", grid_n=24, tol=0.01, seed=501,
                              max_walks=4_000_000)
    assert res["converged"]
    row = ids.index(res["master_id"])
    by_id = {t["conductor_id"]: t["capacitance_farads"] for t in res["terminals"]}
    num = sum(abs(by_id[c] - cap[row, k]) for k, c in enumerate(ids))
    den = sum(abs(cap[row, k]) for k in range(len(ids)))
    assert num / den <= 0.05, (num / den, by_id, cap[row])
