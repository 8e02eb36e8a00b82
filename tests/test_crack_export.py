"""N4 post-processing (paper_2508_04076_b200/crack.py): crack polygons of the split records,
VTK export, connected components of the fractured elements.  CPU only (uses oracle records)."""
import numpy as np
import pytest

import cem_inputs as ci
import oracle
from paper_2508_04076_b200 import crack


def test_decode_covers_the_24_candidates():
    seen = set()
    for k in range(24):
        c, p, q, r, t = crack.decode(k)
        assert sorted([c, p, q, r]) == [0, 1, 2, 3] and p < q and t == k % 2
        seen.add((c, p, q, t))
    assert len(seen) == 24


@pytest.mark.parametrize("k", range(24))
def test_polygon_geometry(k):
    """Pattern I: the side midpoints of the skew quadrilateral c-p-r-q form a parallelogram
    normal to (X_q - X_p) x (X_r - X_c); pattern II: a triangle parallel to face pqr."""
    rng = np.random.default_rng(k)
    X = np.eye(4, 3, -1) + 0.1 * rng.standard_normal((4, 3))
    (poly,) = crack.crack_polygons(X, np.array([[0, 1, 2, 3]]), [0], [k])
    c, p, q, r, t = crack.decode(k)
    if t == 0:
        m = np.cross(X[q] - X[p], X[r] - X[c])
        assert poly.shape == (4, 3)
        assert np.allclose(poly[0] + poly[2], poly[1] + poly[3], atol=1e-15)
    else:
        m = np.cross(X[q] - X[p], X[r] - X[p])
        assert poly.shape == (3, 3)
    for a in range(len(poly)):
        d = poly[(a + 1) % len(poly)] - poly[a]
        assert abs(d @ m) <= 1e-12 * np.linalg.norm(d) * np.linalg.norm(m)


def test_vtk_round_trip(tmp_path):
    p = ci.config(0)
    o = oracle.Oracle(p)
    o.run(120, 1)
    r = o.records()
    polys = crack.crack_polygons(p.X, p.tets, r.elem, r.cand)
    f = tmp_path / "crack.vtk"
    crack.write_crack_vtk(f, polys, r.G)
    back = crack.read_crack_vtk(f)
    assert len(back) == len(polys) == r.elem.size > 0
    for a, b in zip(polys, back):
        assert np.array_equal(a, b)


def test_components():
    # a column of cells: tets of one cube share faces (Kuhn subdivision), neighbouring cubes too
    X, T, _ = ci.kuhn_lattice((4, 1, 1), (4.0, 1.0, 1.0), 0, jitter=0.0)
    n, lab = crack.crack_components(T, np.arange(T.shape[0]))
    assert n == 1 and np.all(lab == 0)
    # first and last cube only: two components
    el = np.concatenate([np.arange(6), np.arange(18, 24)])
    n, lab = crack.crack_components(T, el)
    assert n == 2 and len(set(lab[:6])) == 1 and len(set(lab[6:])) == 1 and lab[0] != lab[-1]
    assert crack.crack_components(T, [])[0] == 0
