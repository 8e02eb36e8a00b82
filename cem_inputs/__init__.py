"""Seeded synthetic input generators shared by the oracle tests and the product path.

This module holds NONE of the method's arithmetic (no strain, stress, force, mass,
energy-release-rate or time-integration formula).  It only builds meshes and load
descriptions: node coordinates, tet connectivity, per-tet state / Gc, the list of
boundary triangles that carry a traction and the prescribed-velocity nodes.  Both
`oracle/` and `paper_2508_04076_b200/` consume its output; neither imports the other.

Recipe:
  * Kuhn lattice: cube (i,j,k) -> 6 tets, one per axis permutation in lexicographic
    order (x,y,z),(x,z,y),(y,x,z),(y,z,x),(z,x,y),(z,y,x); each tet follows the vertex
    path (0,0,0) -> +e_p0 -> +e_p1 -> (1,1,1); for odd permutations local vertices 2
    and 3 are swapped so every tet has positive orientation.
  * ids: tet = 6*cell + perm, cell = i + nx*(j + ny*k), node = i + (nx+1)*(j + (ny+1)*k).
  * jitter: component c of node v moves by (2U-1)*0.05*h_c with
    U = (splitmix64(splitmix64(seed) ^ (3v+c)) >> 11) * 2^-53; components on a boundary
    plane (lattice index 0 or n_c) are not moved.
  * notch: cells (i < nx/2, j = ny/2 - 1, all k) start inactive (state 0).
  * pre-damage (config 3): tet t gets Gc_e = 0 iff
    (splitmix64(splitmix64(seed ^ 0xD1B54A32D192ED03) ^ t) >> 11) * 2^-53 < fraction.
  * traction: the boundary triangles of active tets lying on the planes y = 0 and
    y = Ly (lattice j = 0 / j = ny) carry (0, -t, 0) / (0, +t, 0); they are listed in
    ascending (tet id, local face id) order, local face f = the face opposite vertex f.

The paper's own meshes are not available (figures are placeholders, PAPER.md:L1131
lists only counts), so these seeded lattices stand in for its workloads
(PAPER.md:L1118-L1131 Neumann branching plate; PAPER.md:L546-L581 Kalthoff plate).
"""
from __future__ import annotations

from dataclasses import dataclass, field
from typing import Optional

import numpy as np

__all__ = [
    "Problem", "splitmix64", "kuhn_lattice", "notched_plate", "edge_impact_plate",
    "weak_scaling_block", "config", "CONFIGS", "random_tet_mesh", "single_tet",
]

_M64 = np.uint64(0xFFFFFFFFFFFFFFFF)

# permutations of the axes in lexicographic order and their parity
_PERMS = [(0, 1, 2), (0, 2, 1), (1, 0, 2), (1, 2, 0), (2, 0, 1), (2, 1, 0)]
_ODD = [False, True, True, False, False, True]


def splitmix64(x):
    """SplitMix64 finaliser on uint64 arrays (wrap-around arithmetic)."""
    z = np.asarray(x, dtype=np.uint64)
    with np.errstate(over="ignore"):
        z = z + np.uint64(0x9E3779B97F4A7C15)
        z = (z ^ (z >> np.uint64(30))) * np.uint64(0xBF58476D1CE4E5B9)
        z = (z ^ (z >> np.uint64(27))) * np.uint64(0x94D049BB133111EB)
        z = z ^ (z >> np.uint64(31))
    return z


def _unit(seed_word, idx):
    """U in [0,1) from a hashed seed word and an index array: (h >> 11) * 2^-53."""
    h = splitmix64(np.uint64(seed_word) ^ np.asarray(idx, dtype=np.uint64))
    return (h >> np.uint64(11)).astype(np.float64) * (2.0 ** -53)


@dataclass
class Problem:
    """One seeded problem instance (everything the C-ABI `cem_init_mesh` takes)."""
    name: str
    X: np.ndarray                     # [N,3] float64 reference coordinates (m)
    tets: np.ndarray                  # [E,4] int32, positive orientation
    tet_state: np.ndarray             # [E] uint8: 1 active, 0 inactive (notch)
    tet_gc: np.ndarray                # [E] float64 per-element Gc (J/m^2)
    E: float                          # Young's modulus (Pa)
    nu: float                         # Poisson ratio
    rho: float                        # density (kg/m^3)
    Gc: float                         # nominal critical energy release rate (J/m^2)
    tface: np.ndarray                 # [F,3] int32 loaded boundary triangles
    tface_t: np.ndarray               # [F,3] float64 traction on each (Pa)
    vbc_node: np.ndarray              # [B] int32 prescribed-velocity nodes
    vbc_mask: np.ndarray              # [B] uint8 bit0=x bit1=y bit2=z
    vbc_v0: np.ndarray                # [B,3] float64 target velocity (m/s)
    vbc_t0: float = 0.0               # ramp time (s)
    steps: int = 0                    # nominal number of steps of the config
    dt: float = 0.0                   # <= 0: cfl * min altitude / c_d
    cfl: float = 0.5
    gamma: float = 0.5
    cells: tuple = (0, 0, 0)
    dims: tuple = (0.0, 0.0, 0.0)
    node_ijk: Optional[np.ndarray] = None   # [N,3] lattice indices (tests only)
    f_nodal: Optional[np.ndarray] = None    # [N,3] constant nodal point forces (N), or None
    body: tuple = (0.0, 0.0, 0.0)           # uniform body force density b (N/m^3)
    meta: dict = field(default_factory=dict)

    @property
    def n_nodes(self) -> int:
        return int(self.X.shape[0])

    @property
    def n_tets(self) -> int:
        return int(self.tets.shape[0])

    def with_gc(self, gc: float) -> "Problem":
        """Copy with every (non pre-damaged) Gc replaced by `gc`."""
        p = Problem(**{k: getattr(self, k) for k in self.__dataclass_fields__})
        g = np.where(self.tet_gc == 0.0, 0.0, gc)
        p.tet_gc = g.astype(np.float64)
        p.Gc = gc
        return p


def kuhn_lattice(cells, dims, seed, jitter=0.05):
    """Jittered Kuhn lattice. Returns (X [N,3], tets [E,4] int32, node_ijk [N,3])."""
    nx, ny, nz = (int(c) for c in cells)
    Lx, Ly, Lz = (float(d) for d in dims)
    n = np.array([nx, ny, nz])
    ii, jj, kk = np.meshgrid(np.arange(nx + 1), np.arange(ny + 1), np.arange(nz + 1), indexing="ij")
    # node id = i + (nx+1)*(j + (ny+1)*k): order arrays with i fastest
    ijk = np.stack([ii.transpose(2, 1, 0).ravel(), jj.transpose(2, 1, 0).ravel(),
                    kk.transpose(2, 1, 0).ravel()], axis=1).astype(np.int64)
    L = np.array([Lx, Ly, Lz])
    X = ijk.astype(np.float64) * L[None, :] / n[None, :].astype(np.float64)
    if jitter:
        h = L / n
        v = np.arange(ijk.shape[0], dtype=np.uint64)
        s = splitmix64(np.uint64(seed))
        for c in range(3):
            U = _unit(s, np.uint64(3) * v + np.uint64(c))
            d = (2.0 * U - 1.0) * jitter * h[c]
            interior = (ijk[:, c] > 0) & (ijk[:, c] < n[c])
            X[:, c] = X[:, c] + np.where(interior, d, 0.0)
    # tets
    ci, cj, ck = np.meshgrid(np.arange(nx), np.arange(ny), np.arange(nz), indexing="ij")
    ci = ci.transpose(2, 1, 0).ravel(); cj = cj.transpose(2, 1, 0).ravel(); ck = ck.transpose(2, 1, 0).ravel()
    ncell = ci.size
    sx, sy = nx + 1, (nx + 1) * (ny + 1)

    def nid(di, dj, dk):
        return (ci + di) + sx * (cj + dj) + sy * (ck + dk)

    tets = np.empty((ncell, 6, 4), dtype=np.int64)
    for p, perm in enumerate(_PERMS):
        off = [0, 0, 0]
        verts = [nid(0, 0, 0)]
        for ax in perm[:2]:
            off[ax] += 1
            verts.append(nid(*off))
        verts.append(nid(1, 1, 1))
        if _ODD[p]:
            verts[2], verts[3] = verts[3], verts[2]
        tets[:, p, :] = np.stack(verts, axis=1)
    return X, tets.reshape(-1, 4).astype(np.int32), ijk


def hex_lattice(cells, dims, seed, jitter=0.05):
    """Jittered structured hexahedral lattice (same node numbering and jitter as kuhn_lattice).
    Hex = cell (i,j,k), local nodes 0-3 on the k face counter-clockwise from (i,j), 4-7 above.
    Returns (X [N,3], hexes [E,8] int32, node_ijk [N,3])."""
    X, _, ijk = kuhn_lattice(cells, dims, seed, jitter=jitter)
    nx, ny, nz = (int(c) for c in cells)
    ci, cj, ck = np.meshgrid(np.arange(nx), np.arange(ny), np.arange(nz), indexing="ij")
    ci = ci.transpose(2, 1, 0).ravel(); cj = cj.transpose(2, 1, 0).ravel(); ck = ck.transpose(2, 1, 0).ravel()
    sx, sy = nx + 1, (nx + 1) * (ny + 1)

    def nid(di, dj, dk):
        return (ci + di) + sx * (cj + dj) + sy * (ck + dk)

    H = np.stack([nid(0, 0, 0), nid(1, 0, 0), nid(1, 1, 0), nid(0, 1, 0),
                  nid(0, 0, 1), nid(1, 0, 1), nid(1, 1, 1), nid(0, 1, 1)], axis=1)
    return X, H.astype(np.int32), ijk


def hex_block(cells=(12, 8, 4), dims=(0.06, 0.04, 0.02), seed=8, traction=1e6, jitter=0.05, steps=0,
              material=None, gc=np.inf, notch=0.0):
    """Hexahedral block for the ES-H-FEM path: traction +-t on the y faces as
    two triangles per loaded quad face (t A/3 per triangle node).  gc: critical energy release rate
    of every hex (inf: no cracking); notch > 0: the hexes of the middle y layer with x below
    notch * length are inactive (an edge notch across the pulled direction)."""
    mat = dict(E=32e9, nu=0.2, rho=2450.0) if material is None else material
    X, H, ijk = hex_lattice(cells, dims, seed, jitter=jitter)
    ny = int(cells[1])
    faces, tr = [], []
    for jv, sgn in ((0, -1.0), (ny, 1.0)):
        on = ijk[:, 1] == jv
        for e in range(H.shape[0]):
            for quad in ([0, 1, 5, 4], [3, 2, 6, 7]):
                q = H[e, quad]
                if on[q].all():
                    faces += [[q[0], q[1], q[2]], [q[0], q[2], q[3]]]
                    tr += [[0.0, sgn * traction, 0.0]] * 2
    E = H.shape[0]
    state = np.ones(E, np.uint8)
    if notch > 0:
        nx = int(cells[0])
        ci = np.arange(E) % nx
        cj = (np.arange(E) // nx) % ny
        state[(cj == ny // 2) & (ci < int(round(notch * nx)))] = 0
    return Problem(name=f"hex_block_{cells[0]}x{cells[1]}x{cells[2]}", X=X, tets=H,
                   tet_state=state, tet_gc=np.full(E, float(gc)), Gc=float(gc),
                   tface=np.asarray(faces, np.int32).reshape(-1, 3), tface_t=np.asarray(tr, np.float64).reshape(-1, 3),
                   vbc_node=np.zeros(0, np.int32), vbc_mask=np.zeros(0, np.uint8), vbc_v0=np.zeros((0, 3)),
                   steps=steps, cells=tuple(cells), dims=tuple(dims), node_ijk=ijk, **mat)


def _loaded_faces(tets, tet_state, node_ijk, axis, index, traction):
    """Boundary triangles of active tets whose 3 nodes have lattice index `index` on `axis`."""
    E = tets.shape[0]
    faces, owner = [], []
    on = node_ijk[:, axis] == index
    for f in range(4):
        keep = [a for a in range(4) if a != f]
        tri = tets[:, keep]
        hit = on[tri].all(axis=1) & (tet_state == 1)
        idx = np.nonzero(hit)[0]
        faces.append(tri[idx]); owner.append(idx * 4 + f)
    faces = np.concatenate(faces); owner = np.concatenate(owner)
    order = np.argsort(owner, kind="stable")
    faces = faces[order].astype(np.int32)
    t = np.tile(np.asarray(traction, dtype=np.float64), (faces.shape[0], 1))
    return faces, t, owner[order]


def _merge_faces(*parts):
    """Merge (faces, t, owner) lists keeping ascending (tet, local face) order."""
    faces = np.concatenate([p[0] for p in parts]) if parts else np.zeros((0, 3), np.int32)
    t = np.concatenate([p[1] for p in parts]) if parts else np.zeros((0, 3))
    owner = np.concatenate([p[2] for p in parts]) if parts else np.zeros(0, np.int64)
    order = np.argsort(owner, kind="stable")
    return faces[order].astype(np.int32), t[order]


def _cell_of_tet(E):
    return np.arange(E) // 6


def _empty_vbc():
    return (np.zeros(0, np.int32), np.zeros(0, np.uint8), np.zeros((0, 3), np.float64))


CONCRETE = dict(E=32e9, nu=0.2, rho=2450.0, Gc=3.0)
STEEL = dict(E=190e9, nu=0.3, rho=8000.0, Gc=22.2e3)         # PAPER.md:L571 (BASELINE cfg 2)


def notched_plate(cells=(20, 8, 2), dims=(0.1, 0.04, 0.005), seed=0, traction=1e6,
                  notch=True, steps=200, material=CONCRETE, name=None, predamage=0.0,
                  predamage_seed=None, jitter=0.05):
    """Pre-notched plate pulled by +-traction on y=0 / y=Ly."""
    nx, ny, nz = cells
    X, tets, ijk = kuhn_lattice(cells, dims, seed, jitter)
    E = tets.shape[0]
    state = np.ones(E, np.uint8)
    if notch:
        cell = _cell_of_tet(E)
        ci = cell % nx; cj = (cell // nx) % ny
        state[(ci < nx // 2) & (cj == ny // 2 - 1)] = 0
    gc = np.full(E, material["Gc"], np.float64)
    if predamage > 0.0:
        ps = predamage_seed if predamage_seed is not None else seed
        U = _unit(splitmix64(np.uint64(ps) ^ np.uint64(0xD1B54A32D192ED03)), np.arange(E, dtype=np.uint64))
        gc[U < predamage] = 0.0
    bottom = _loaded_faces(tets, state, ijk, 1, 0, (0.0, -traction, 0.0))
    top = _loaded_faces(tets, state, ijk, 1, ny, (0.0, traction, 0.0))
    tface, tface_t = _merge_faces(bottom, top)
    vb = _empty_vbc()
    return Problem(name=name or f"notched_plate{tuple(cells)}", X=X, tets=tets, tet_state=state,
                   tet_gc=gc, E=material["E"], nu=material["nu"], rho=material["rho"],
                   Gc=material["Gc"], tface=tface, tface_t=tface_t, vbc_node=vb[0],
                   vbc_mask=vb[1], vbc_v0=vb[2], vbc_t0=0.0, steps=steps, cells=tuple(cells),
                   dims=tuple(dims), node_ijk=ijk)


def edge_impact_plate(cells=(200, 100, 9), dims=(0.2, 0.1, 0.009), seed=2, v0=16.5, t0=1e-6,
                      steps=2000, material=STEEL, name=None):
    """Kalthoff-Winkler stand-in: two edge notches, v_x ramp on x=0.

    Notches: cells i < nx/4 at j = ny/4 - 1 and j = 3ny/4 (y ~ 0.025 / 0.075 for ny=100).
    Prescribed v_x (ramp v = t/t0 v0) on x=0 nodes with
    ny/4 <= j <= 3ny/4.
    """
    nx, ny, nz = cells
    X, tets, ijk = kuhn_lattice(cells, dims, seed)
    E = tets.shape[0]
    state = np.ones(E, np.uint8)
    cell = _cell_of_tet(E)
    ci = cell % nx; cj = (cell // nx) % ny
    state[(ci < nx // 4) & ((cj == ny // 4 - 1) | (cj == (3 * ny) // 4))] = 0
    gc = np.full(E, material["Gc"], np.float64)
    sel = np.nonzero((ijk[:, 0] == 0) & (ijk[:, 1] >= ny // 4) & (ijk[:, 1] <= (3 * ny) // 4))[0]
    vbc_node = sel.astype(np.int32)
    vbc_mask = np.full(sel.size, 1, np.uint8)
    vbc_v0 = np.zeros((sel.size, 3)); vbc_v0[:, 0] = v0
    return Problem(name=name or f"edge_impact{tuple(cells)}", X=X, tets=tets, tet_state=state,
                   tet_gc=gc, E=material["E"], nu=material["nu"], rho=material["rho"],
                   Gc=material["Gc"], tface=np.zeros((0, 3), np.int32), tface_t=np.zeros((0, 3)),
                   vbc_node=vbc_node, vbc_mask=vbc_mask, vbc_v0=vbc_v0, vbc_t0=t0, steps=steps,
                   cells=tuple(cells), dims=tuple(dims), node_ijk=ijk)


CONCRETE_CT = dict(E=36e9, nu=0.18, rho=2400.0, Gc=65.0)  # PAPER.md:L1343 (Ozbolt et al. concrete)


def compact_tension(cells=(60, 60, 12), dims=(0.2, 0.2, 0.04), seed=5, v0=3.318, t0=100e-6,
                    slot_depth=0.4, steps=1250, material=CONCRETE_CT, name=None):
    """Dynamic compact tension stand-in.

    The paper's geometry figure is missing; approximated as a W x H x B block with a vertical
    slot (two cells wide, inactive) cut from the top face to depth slot_depth * H at mid-width.
    The slot's right face (node column i = nx/2 + 1) is driven in x by the ramp v = (t/t0) v0
    (t0 = 100 us, v0 = 1.375 / 3.318 / 3.993 m/s), its left face
    (i = nx/2 - 1) is held at v_x = 0.  The crack grows from the slot tip towards y = 0.
    """
    nx, ny, nz = cells
    X, tets, ijk = kuhn_lattice(cells, dims, seed)
    E = tets.shape[0]
    cell = _cell_of_tet(E)
    ci = cell % nx; cj = (cell // nx) % ny
    depth = max(1, int(round(slot_depth * ny)))
    state = np.ones(E, np.uint8)
    state[((ci == nx // 2 - 1) | (ci == nx // 2)) & (cj >= ny - depth)] = 0
    gc = np.full(E, material["Gc"], np.float64)
    on_slot = ijk[:, 1] >= ny - depth
    right = np.nonzero(on_slot & (ijk[:, 0] == nx // 2 + 1))[0]
    left = np.nonzero(on_slot & (ijk[:, 0] == nx // 2 - 1))[0]
    vbc_node = np.concatenate([left, right]).astype(np.int32)
    order = np.argsort(vbc_node, kind="stable")
    vbc_node = vbc_node[order]
    vbc_v0 = np.zeros((vbc_node.size, 3))
    vbc_v0[:, 0] = np.concatenate([np.zeros(left.size), np.full(right.size, v0)])[order]
    vbc_mask = np.full(vbc_node.size, 1, np.uint8)
    return Problem(name=name or f"compact_tension{tuple(cells)}_v{v0}", X=X, tets=tets, tet_state=state,
                   tet_gc=gc, E=material["E"], nu=material["nu"], rho=material["rho"], Gc=material["Gc"],
                   tface=np.zeros((0, 3), np.int32), tface_t=np.zeros((0, 3)), vbc_node=vbc_node,
                   vbc_mask=vbc_mask, vbc_v0=vbc_v0, vbc_t0=t0, steps=steps, cells=tuple(cells),
                   dims=tuple(dims), node_ijk=ijk)


def weak_scaling_block(P=1, cells_per_rank=(100, 100, 17), h=1e-3, seed=3, predamage=0.005,
                       steps=1000):
    """Config 3: (100P) x 100 x 17 cells, h = 1 mm, no notch, 0.5% pre-damaged tets (Gc_e = 0)."""
    nx, ny, nz = cells_per_rank
    cells = (nx * P, ny, nz)
    dims = (cells[0] * h, ny * h, nz * h)
    return notched_plate(cells=cells, dims=dims, seed=seed, notch=False, steps=steps,
                         name=f"weak_block_P{P}{tuple(cells)}", predamage=predamage,
                         predamage_seed=seed)


def config(k: int, P: int = 1) -> Problem:
    """BASELINE.json configs[k] as a seeded synthetic Problem."""
    if k == 0:
        return notched_plate((20, 8, 2), seed=0, steps=200, name="cfg0")
    if k == 1:
        return notched_plate((120, 48, 6), seed=1, steps=5000, name="cfg1")
    if k == 2:
        return edge_impact_plate(name="cfg2")
    if k == 3:
        p = weak_scaling_block(P=P)
        p.name = f"cfg3_P{P}"
        return p
    if k == 4:
        return notched_plate((400, 160, 20), seed=4, steps=10000, name="cfg4")
    if k in (5, 6, 7):  # N2: dynamic compact tension, the paper's three loading rates
        v0 = {5: 1.375, 6: 3.318, 7: 3.993}[k]
        return compact_tension(v0=v0, name=f"cfg{k}_ct_v{v0}")
    raise ValueError(k)


CONFIGS = {0: "cfg0", 1: "cfg1", 2: "cfg2", 3: "cfg3", 4: "cfg4", 5: "cfg5_ct", 6: "cfg6_ct", 7: "cfg7_ct"}


def single_tet(L=1.0):
    """The unit right tet scaled by L (used by closed-form pins)."""
    X = np.array([[0, 0, 0], [L, 0, 0], [0, L, 0], [0, 0, L]], dtype=np.float64)
    tets = np.array([[0, 1, 2, 3]], dtype=np.int32)
    return X, tets


def random_tet_mesh(seed, n_cells=(2, 2, 1), jitter=0.2):
    """Small strongly-jittered Kuhn mesh for brute-force tests."""
    X, tets, ijk = kuhn_lattice(n_cells, (1.0, 1.0, 1.0), seed, jitter=jitter)
    return X, tets, ijk


def fan_mesh(m=40, r=0.01, h=0.01, seed=0, jitter=0.2):
    """m tets around one axis edge (0,0,-h)-(0,0,h) with a ring of m nodes near radius r: the axis
    edge and its two end nodes have valence m (tests the ELL widths past 8/24).  Tet i =
    (bottom, top, ring_i, ring_{i+1}), positively oriented for a counter-clockwise ring; seeded
    jitter of the ring radii, angles (< half a sector) and heights breaks the symmetry."""
    rng = np.random.default_rng(seed)
    th = 2.0 * np.pi * (np.arange(m) + jitter * rng.uniform(-0.5, 0.5, m)) / m
    rr = r * (1.0 + jitter * rng.uniform(-0.5, 0.5, m))
    z = h * jitter * rng.uniform(-0.5, 0.5, m)
    X = np.concatenate([[[0.0, 0.0, -h], [0.0, 0.0, h]], np.stack([rr * np.cos(th), rr * np.sin(th), z], 1)])
    T = np.array([[0, 1, 2 + i, 2 + (i + 1) % m] for i in range(m)], np.int32)
    return X, T


def make_problem(X, tets, E=32e9, nu=0.2, rho=2450.0, Gc=3.0, tet_state=None, tet_gc=None,
                 tface=None, tface_t=None, vbc=None, dt=0.0, name="custom", steps=0):
    """Wrap raw arrays into a Problem (tests)."""
    En = tets.shape[0]
    st = np.ones(En, np.uint8) if tet_state is None else np.asarray(tet_state, np.uint8)
    gc = np.full(En, Gc, np.float64) if tet_gc is None else np.asarray(tet_gc, np.float64)
    tf = np.zeros((0, 3), np.int32) if tface is None else np.asarray(tface, np.int32)
    tt = np.zeros((0, 3)) if tface_t is None else np.asarray(tface_t, np.float64)
    if vbc is None:
        vn, vm, vv, t0 = np.zeros(0, np.int32), np.zeros(0, np.uint8), np.zeros((0, 3)), 0.0
    else:
        vn, vm, vv, t0 = vbc
    return Problem(name=name, X=np.ascontiguousarray(X, np.float64),
                   tets=np.ascontiguousarray(tets, np.int32), tet_state=st, tet_gc=gc,
                   E=E, nu=nu, rho=rho, Gc=Gc, tface=tf, tface_t=tt,
                   vbc_node=np.asarray(vn, np.int32), vbc_mask=np.asarray(vm, np.uint8),
                   vbc_v0=np.asarray(vv, np.float64).reshape(-1, 3), vbc_t0=float(t0),
                   steps=steps, dt=dt)
