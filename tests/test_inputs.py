"""Seeded input generator (cem_inputs): entity counts and mesh validity.

Counts: BASELINE.json configs[0] states 1920 tets / 567 nodes; the Kuhn-lattice edge
count is nx ny nz * 7 (cube edges shared) closed form checked by brute force.
"""
import numpy as np
import pytest

import cem_inputs as ci


def kuhn_edge_count(nx, ny, nz):
    # axis edges + face diagonals (one per face) + one body diagonal per cell
    axis = nx * (ny + 1) * (nz + 1) + (nx + 1) * ny * (nz + 1) + (nx + 1) * (ny + 1) * nz
    faces = nx * ny * (nz + 1) + nx * (ny + 1) * nz + (nx + 1) * ny * nz
    return axis + faces + nx * ny * nz


def signed_volumes(X, T):
    d1 = X[T[:, 1]] - X[T[:, 0]]; d2 = X[T[:, 2]] - X[T[:, 0]]; d3 = X[T[:, 3]] - X[T[:, 0]]
    return np.einsum("ij,ij->i", d1, np.cross(d2, d3)) / 6.0


def unique_edges(T):
    pairs = np.concatenate([np.sort(T[:, [p, q]], axis=1) for p, q in
                            [(0, 1), (0, 2), (0, 3), (1, 2), (1, 3), (2, 3)]])
    return np.unique(pairs, axis=0)


@pytest.mark.parametrize("k,nodes,tets,edges", [(0, 567, 1920, 2918), (1, 41503, 207360, 262398)])
def test_config_counts(k, nodes, tets, edges):
    p = ci.config(k)
    assert p.n_nodes == nodes and p.n_tets == tets
    assert unique_edges(p.tets).shape[0] == edges == kuhn_edge_count(*p.cells)


def test_config3_counts():
    p = ci.config(3)
    assert (p.n_tets, p.n_nodes) == (1020000, 183618)
    assert kuhn_edge_count(*p.cells) == 1230417
    frac = (p.tet_gc == 0).mean()
    assert 0.004 < frac < 0.006          # 0.5 % pre-damaged (BASELINE.json configs[3])
    assert (p.tet_state == 1).all()      # no notch


@pytest.mark.parametrize("cells", [(3, 2, 2), (6, 5, 4)])
def test_edge_count_formula_bruteforce(cells):
    X, T, _ = ci.kuhn_lattice(cells, (1, 1, 1), seed=7)
    assert unique_edges(T).shape[0] == kuhn_edge_count(*cells)


def test_positive_volumes_and_total_volume():
    for k in (0, 1):
        p = ci.config(k)
        V = signed_volumes(p.X, p.tets)
        assert V.min() > 0
        assert abs(V.sum() - np.prod(p.dims)) < 1e-12 * np.prod(p.dims)


def test_jitter_bounds_and_boundary_planes():
    p = ci.config(0)
    h = np.array(p.dims) / np.array(p.cells)
    lattice = p.node_ijk * h[None, :]
    d = p.X - lattice
    assert np.all(np.abs(d) <= 0.05 * h[None, :] * (1 + 1e-12))
    on_b = (p.node_ijk == 0) | (p.node_ijk == np.array(p.cells)[None, :])
    assert np.all(d[on_b] == 0.0)
    assert np.abs(d[~on_b]).min() > 0       # interior components really move


def test_notch_and_loads():
    p = ci.config(0)
    nx, ny, nz = p.cells
    assert (p.tet_state == 0).sum() == (nx // 2) * nz * 6
    # loaded triangles: 2 per boundary cell face on y=0 and y=Ly
    assert p.tface.shape[0] == 2 * 2 * nx * nz
    y = p.node_ijk[p.tface][:, :, 1]
    assert np.all((y == 0).all(axis=1) | (y == ny).all(axis=1))
    ty = p.tface_t[:, 1]
    assert np.all(np.where((y == 0).all(axis=1), ty == -1e6, ty == 1e6))


def test_seeded_and_deterministic():
    a = ci.config(0); b = ci.config(0)
    assert np.array_equal(a.X, b.X) and np.array_equal(a.tets, b.tets)
    c = ci.notched_plate(seed=1)
    assert not np.array_equal(a.X, c.X)


def test_edge_impact_plate_small():
    p = ci.edge_impact_plate(cells=(20, 12, 2), dims=(0.02, 0.012, 0.002), steps=10)
    assert p.vbc_node.size == (12 * 3 // 4 - 12 // 4 + 1) * 3
    assert np.all(p.X[p.vbc_node, 0] == 0.0)
    assert (p.tet_state == 0).sum() == 2 * (20 // 4) * 2 * 6


def test_compact_tension_small():
    """N2 stand-in: a two-cell slot from the top to 40 % depth; right slot face driven in x, left held."""
    nx, ny, nz = 16, 20, 3
    p = ci.compact_tension(cells=(nx, ny, nz), dims=(0.16, 0.2, 0.03), v0=3.318)
    depth = 8
    assert (p.tet_state == 0).sum() == 2 * depth * nz * 6
    assert p.vbc_node.size == 2 * (depth + 1) * (nz + 1)
    assert np.all(np.diff(p.vbc_node) > 0)
    assert np.all(p.vbc_mask == 1)
    ijk = p.node_ijk[p.vbc_node]
    assert set(np.unique(ijk[:, 0])) == {nx // 2 - 1, nx // 2 + 1}
    assert np.all(p.vbc_v0[ijk[:, 0] == nx // 2 + 1, 0] == 3.318)
    assert np.all(p.vbc_v0[ijk[:, 0] == nx // 2 - 1] == 0.0)
    assert p.vbc_t0 == 100e-6 and p.E == 36e9 and p.nu == 0.18 and p.Gc == 65.0
