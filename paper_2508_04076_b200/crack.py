"""Crack-surface export and branch detection (SPEC.md write_vtk_snapshot,
acceptance criterion 3) -- post-processing of the split records, off the hot path.

A record (element e, candidate k) names the crack pattern the criterion chose (R7):
k = 6c + 2f + t, corner c, front {p, q} among the other nodes o0 < o1 < o2 as (o0,o1), (o0,o2),
(o1,o2), r the remaining node;
  t = 0, pattern I:  quadrilateral through the midpoints of c-p, c-q, q-r, p-r   (Fig. 5);
  t = 1, pattern II: triangle through the midpoints of c-p, c-q, c-r.
"""
from __future__ import annotations

import numpy as np


def decode(k: int):
    """(c, p, q, r, t) of candidate k."""
    c, f, t = k // 6, (k % 6) // 2, k & 1
    o = [b for b in range(4) if b != c]
    p, q, r = o[1 if f == 2 else 0], o[1 if f == 0 else 2], o[2 - f]
    return c, p, q, r, t


def crack_polygons(X, tets, rec_elem, rec_cand, u=None):
    """Polygons of the recorded splits: list of (m, 3) vertex arrays (m = 4 or 3), in the
    reference configuration, or the deformed one X + u when u is given."""
    P = np.asarray(X, np.float64) if u is None else np.asarray(X, np.float64) + np.asarray(u, np.float64)
    T = np.asarray(tets)
    polys = []
    for e, k in zip(np.asarray(rec_elem), np.asarray(rec_cand)):
        c, p, q, r, t = decode(int(k))
        x = P[T[int(e)]]
        mid = lambda a, b: 0.5 * (x[a] + x[b])  # noqa: E731
        if t == 0:
            polys.append(np.array([mid(c, p), mid(c, q), mid(q, r), mid(p, r)]))
        else:
            polys.append(np.array([mid(c, p), mid(c, q), mid(c, r)]))
    return polys


def write_crack_vtk(path, polys, values=None, name="G"):
    """Legacy ASCII VTK POLYDATA with one polygon per split (optional per-polygon scalar)."""
    npts = sum(len(p) for p in polys)
    with open(path, "w") as f:
        f.write("# vtk DataFile Version 3.0\ncrack surface (CEM split records)\nASCII\nDATASET POLYDATA\n")
        f.write(f"POINTS {npts} double\n")
        for p in polys:
            for v in p:
                f.write(f"{v[0]:.17g} {v[1]:.17g} {v[2]:.17g}\n")
        f.write(f"POLYGONS {len(polys)} {npts + len(polys)}\n")
        i = 0
        for p in polys:
            f.write(" ".join([str(len(p))] + [str(i + j) for j in range(len(p))]) + "\n")
            i += len(p)
        if values is not None:
            f.write(f"CELL_DATA {len(polys)}\nSCALARS {name} double 1\nLOOKUP_TABLE default\n")
            for v in values:
                f.write(f"{float(v):.17g}\n")


def read_crack_vtk(path):
    """Inverse of write_crack_vtk (tests): list of (m, 3) arrays."""
    lines = open(path).read().split("\n")
    i = next(j for j, s in enumerate(lines) if s.startswith("POINTS"))
    n = int(lines[i].split()[1])
    pts = np.array([[float(v) for v in lines[i + 1 + j].split()] for j in range(n)])
    i = next(j for j, s in enumerate(lines) if s.startswith("POLYGONS"))
    m = int(lines[i].split()[1])
    out = []
    for j in range(m):
        ids = [int(v) for v in lines[i + 1 + j].split()]
        out.append(pts[ids[1:1 + ids[0]]])
    return out


def crack_components(tets, rec_elem):
    """Connected components of the fractured elements, two split tets being adjacent when
    they share a face (SPEC.md acceptance criterion 3: 'connectedness computed on the
    fractured-element adjacency graph').  Returns (n_components, label per record)."""
    T = np.asarray(tets)
    el = np.asarray(rec_elem, np.int64)
    if el.size == 0:
        return 0, np.zeros(0, np.int64)
    parent = list(range(el.size))

    def find(a):
        while parent[a] != a:
            parent[a] = parent[parent[a]]
            a = parent[a]
        return a

    faces = {}
    for i, e in enumerate(el):
        v = T[e]
        for f in range(4):
            key = tuple(sorted(int(v[a]) for a in range(4) if a != f))
            j = faces.setdefault(key, i)
            if j != i:
                ra, rb = find(i), find(j)
                if ra != rb:
                    parent[max(ra, rb)] = min(ra, rb)
    roots = np.array([find(i) for i in range(el.size)])
    _, lab = np.unique(roots, return_inverse=True)
    return int(lab.max()) + 1, lab
