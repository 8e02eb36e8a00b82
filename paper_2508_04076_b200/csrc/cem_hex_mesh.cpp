// cem_hex_mesh.cpp -- host preprocessing of the ES-H-FEM path on trilinear hexahedra (SURVEY.md §8(f)
// N3; PAPER.md:L311-L338 eq:hex_strain_discretization, L368-L390 eq:hex_fint_discretization):
// validation, mean-gradient geometry, the 12-edge topology, incidence tables, lumped mass,
// external force and time step.  Readings R23-R26; every expression rounds as
// written (-ffp-contract=off) in the association order DESIGN.md §5 fixes for hexes.
#include <algorithm>
#include <cmath>
#include <numeric>

#include "cem_internal.h"

namespace cem {

namespace {

// reference coordinates of the local nodes (bottom face 0-3 counter-clockwise, top face 4-7)
const double kXi[8][3] = {{-1, -1, -1}, {1, -1, -1}, {1, 1, -1}, {-1, 1, -1},
                          {-1, -1, 1},  {1, -1, 1},  {1, 1, 1},  {-1, 1, 1}};
const int kFace[6][4] = {{0, 1, 2, 3}, {4, 5, 6, 7}, {0, 1, 5, 4}, {1, 2, 6, 5}, {2, 3, 7, 6}, {3, 0, 4, 7}};

struct W3 {
    double x, y, z;
};
inline W3 wsub(W3 a, W3 b) { return {a.x - b.x, a.y - b.y, a.z - b.z}; }
inline double wdot(W3 a, W3 b) { return (a.x * b.x + a.y * b.y) + a.z * b.z; }
inline W3 wcross(W3 a, W3 b) { return {a.y * b.z - a.z * b.y, a.z * b.x - a.x * b.z, a.x * b.y - a.y * b.x}; }

// dN_i/dxi at p: N_i = (1 + xi xi_i)(1 + eta eta_i)(1 + zeta zeta_i) / 8
inline void dN(const double *p, int i, double *g) {
    const double a = 1.0 + p[0] * kXi[i][0], b = 1.0 + p[1] * kXi[i][1], c = 1.0 + p[2] * kXi[i][2];
    g[0] = (kXi[i][0] * b * c) / 8.0;
    g[1] = (a * kXi[i][1] * c) / 8.0;
    g[2] = (a * b * kXi[i][2]) / 8.0;
}
// the Jacobian's columns dx/dxi_c = sum_i x_i dN_i/dxi_c (i ascending)
inline void jac_cols(const double *X8, const double *p, W3 &c0, W3 &c1, W3 &c2) {
    double J[3][3] = {{0, 0, 0}, {0, 0, 0}, {0, 0, 0}};
    for (int i = 0; i < 8; ++i) {
        double g[3];
        dN(p, i, g);
        for (int r = 0; r < 3; ++r)
            for (int c = 0; c < 3; ++c) J[r][c] = J[r][c] + X8[3 * i + r] * g[c];
    }
    c0 = {J[0][0], J[1][0], J[2][0]};
    c1 = {J[0][1], J[1][1], J[2][1]};
    c2 = {J[0][2], J[1][2], J[2][2]};
}

}  // namespace

// Element geometry (R23, R24): V = sum over the 2x2x2 Gauss points of det J, mean gradients
// grad_a = (sum_g cof(J_g) dN_a/dxi) / V with (cof dN)_r = ((c1 x c2)_r dN_0 + (c2 x c0)_r dN_1)
// + (c0 x c1)_r dN_2.  Returns false unless det J > 0 at the 8 corners.
bool hex_geometry(const double *X8, double &V, double *grad) {
    for (int k = 0; k < 8; ++k) {
        W3 c0, c1, c2;
        jac_cols(X8, kXi[k], c0, c1, c2);
        if (!(wdot(c0, wcross(c1, c2)) > 0.0)) return false;
    }
    const double gp = 1.0 / std::sqrt(3.0);
    double vol = 0.0, acc[8][3];
    for (int a = 0; a < 8; ++a) acc[a][0] = acc[a][1] = acc[a][2] = 0.0;
    for (int k = 0; k < 8; ++k) {
        const double p[3] = {kXi[k][0] * gp, kXi[k][1] * gp, kXi[k][2] * gp};
        W3 c0, c1, c2;
        jac_cols(X8, p, c0, c1, c2);
        const W3 r0 = wcross(c1, c2), r1 = wcross(c2, c0), r2 = wcross(c0, c1);
        vol = vol + wdot(c0, r0);
        const double R0[3] = {r0.x, r0.y, r0.z}, R1[3] = {r1.x, r1.y, r1.z}, R2[3] = {r2.x, r2.y, r2.z};
        for (int a = 0; a < 8; ++a) {
            double g[3];
            dN(p, a, g);
            for (int r = 0; r < 3; ++r) acc[a][r] = acc[a][r] + ((R0[r] * g[0] + R1[r] * g[1]) + R2[r] * g[2]);
        }
    }
    if (!(vol > 0.0)) return false;
    const double inv = 1.0 / vol;
    for (int a = 0; a < 8; ++a)
        for (int r = 0; r < 3; ++r) grad[3 * a + r] = acc[a][r] * inv;
    V = vol;
    return true;
}

cem_status build_hex_host(const cem_mesh_in *m, const cem_material *mat, const cem_load_in *ld, const cem_opts *o,
                          HexHost &h, std::string &err) {
    if (!m || !mat || !m->X || !m->tets || m->n_nodes <= 0 || m->n_tets <= 0) {
        err = "cem_init_mesh: empty mesh or NULL array";
        return CEM_EINVAL;
    }
    if (!(mat->E > 0) || !(mat->nu > -1.0 && mat->nu < 0.5) || !(mat->rho > 0)) {
        err = "cem_init_mesh: material needs E > 0, -1 < nu < 0.5, rho > 0";
        return CEM_EINVAL;
    }
    const double gamma = o && o->gamma > 0 ? o->gamma : 0.5;
    const double cfl = o && o->cfl > 0 ? o->cfl : 0.5;
    if (gamma > 1.0) {
        err = "cem_init_mesh: gamma must be in (0, 1]";
        return CEM_EINVAL;
    }
    const int64_t N = m->n_nodes, E = m->n_tets;
    if (E > ((int64_t)1 << 31) / 96 - 64 || N >= ((int64_t)1 << 31)) {
        err = "hex mesh too large for one context (E < 22M)";
        return CEM_EINVAL;
    }
    h.N = N;
    h.E = E;
    h.hex.assign(m->tets, m->tets + 8 * E);
    h.state.resize(E);
    for (int64_t e = 0; e < E; ++e) h.state[e] = m->tet_state ? (m->tet_state[e] != 0) : 1;
    for (int64_t i = 0; i < 8 * E; ++i)
        if (h.hex[i] < 0 || h.hex[i] >= N) {
            err = "hex " + std::to_string(i / 8) + ": node index out of range";
            return CEM_ETOPOLOGY;
        }
    for (int64_t e = 0; e < E; ++e)
        for (int a = 0; a < 8; ++a)
            for (int b = 0; b < a; ++b)
                if (h.hex[8 * e + a] == h.hex[8 * e + b]) {
                    err = "hex " + std::to_string(e) + ": repeated node";
                    return CEM_ETOPOLOGY;
                }
    for (int64_t i = 0; i < 3 * N; ++i)
        if (!std::isfinite(m->X[i])) {
            err = "node " + std::to_string(i / 3) + ": non-finite coordinate";
            return CEM_EINVAL;
        }
    // ---------------------------------------------------------------- geometry
    h.V.assign(E, 0.0);
    h.grad.assign(24 * E, 0.0);
    int64_t bad = -1;
#pragma omp parallel for schedule(static)
    for (int64_t e = 0; e < E; ++e) {
        double X8[24];
        for (int a = 0; a < 8; ++a)
            for (int c = 0; c < 3; ++c) X8[3 * a + c] = m->X[3 * (int64_t)h.hex[8 * e + a] + c];
        double V;
        if (!hex_geometry(X8, V, h.grad.data() + 24 * e)) {
#pragma omp critical
            bad = bad < 0 ? e : std::min(bad, e);
            continue;
        }
        h.V[e] = V;
    }
    if (bad >= 0) {
        err = "hex " + std::to_string(bad) + ": non-positive Jacobian at a corner";
        return CEM_ENEGVOL;
    }
    // ---------------------------------------------------------------- edges (R28)
    // every local node pair of every hex (28, pair index kHexPair) as a (min, max) key: the pairs that
    // are hex edges of some hex first (the mesh's smoothing domains, edges [0, S_h)), then the face
    // and body diagonals only remainder tets use; each group sorted by key.  Incidence entries
    // (e << 5) | pair in ascending hex id.
    std::vector<std::pair<uint64_t, int64_t>> k(28 * E);
    for (int64_t e = 0; e < E; ++e)
        for (int a = 0; a < 8; ++a)
            for (int b = a + 1; b < 8; ++b) {
                uint64_t i = (uint32_t)h.hex[8 * e + a], j = (uint32_t)h.hex[8 * e + b];
                const uint64_t key = std::min(i, j) << 32 | std::max(i, j);
                const int pj = kHexPair[a][b];
                k[28 * e + pj] = {key | (kHexEdgeOfPair[pj] >= 0 ? 0 : (uint64_t)1 << 63), 28 * e + pj};
            }
    {  // a pair that is a hex edge anywhere is a hex edge everywhere (conforming meshes: never both)
        std::vector<uint64_t> he;
        he.reserve(12 * E);
        for (auto &x : k)
            if (!(x.first >> 63)) he.push_back(x.first);
        std::sort(he.begin(), he.end());
        for (auto &x : k)
            if (x.first >> 63 && std::binary_search(he.begin(), he.end(), x.first & ~((uint64_t)1 << 63)))
                x.first &= ~((uint64_t)1 << 63);
    }
    std::sort(k.begin(), k.end());
    h.pair.resize(28 * E);
    h.eedge.resize(12 * E);
    h.edge_off.clear();
    h.edge_inc.clear();
    int64_t S = 0, S_h = 0;
    for (size_t i = 0; i < k.size(); ++i) {
        if (i == 0 || k[i].first != k[i - 1].first) {
            h.edge_off.push_back((int32_t)h.edge_inc.size());
            ++S;
            if (!(k[i].first >> 63)) S_h = S;
        }
        const int64_t e = k[i].second / 28, pj = k[i].second % 28;
        h.pair[(size_t)pj * E + e] = (int32_t)(S - 1);             // [28][E]
        h.edge_inc.push_back((int32_t)((e << 5) | pj));            // ascending hex id within an edge
    }
    h.edge_off.push_back((int32_t)h.edge_inc.size());
    for (int64_t e = 0; e < E; ++e)
        for (int l = 0; l < 12; ++l) h.eedge[(size_t)l * E + e] = h.pair[(size_t)kHexPair[kHexEdgeP[l]][kHexEdgeQ[l]] * E + e];
    h.S = S;
    h.S_h = S_h;
    h.gc.resize(4 * E);  // hexes, then the remainder tets E + 3e + i (the parent's Gc)
    for (int64_t e = 0; e < E; ++e) {
        h.gc[e] = m->tet_gc ? m->tet_gc[e] : mat->Gc;
        for (int i = 0; i < 3; ++i) h.gc[E + 3 * e + i] = h.gc[e];
    }
    // node incidences 8e + a in ascending e
    h.node_off.assign(N + 1, 0);
    for (int64_t i = 0; i < 8 * E; ++i) h.node_off[h.hex[i] + 1]++;
    for (int64_t n = 0; n < N; ++n) h.node_off[n + 1] += h.node_off[n];
    h.node_ent.resize(8 * E);
    {
        std::vector<int32_t> fill(h.node_off.begin(), h.node_off.end() - 1);
        for (int64_t e = 0; e < E; ++e)
            for (int a = 0; a < 8; ++a) h.node_ent[fill[h.hex[8 * e + a]]++] = (int32_t)(8 * e + a);
    }
    // ---------------------------------------------------------------- material, mass, Vhat
    h.rho = mat->rho;
    h.lam = mat->E * mat->nu / ((1.0 + mat->nu) * (1.0 - 2.0 * mat->nu));
    h.mu = mat->E / (2.0 * (1.0 + mat->nu));
    h.l2m = h.lam + 2.0 * h.mu;
    h.gamma = gamma;
    h.mass.assign(N, 0.0);
    for (int64_t n = 0; n < N; ++n) {  // R24: sum_{active e} (rho V_e)/8 in ascending e
        double acc = 0.0;
        for (int32_t j = h.node_off[n]; j < h.node_off[n + 1]; ++j) {
            const int32_t e = h.node_ent[j] >> 3;
            if (h.state[e]) acc = acc + (h.rho * h.V[e]) / 8.0;
        }
        h.mass[n] = acc;
    }
    // ---------------------------------------------------------------- external force, Dirichlet
    h.fext.assign(3 * N, 0.0);
    h.nflag.assign(N, 0);
    h.dir_v0.assign(3 * N, 0.0);
    if (ld && (ld->body[0] != 0.0 || ld->body[1] != 0.0 || ld->body[2] != 0.0))
        for (int64_t n = 0; n < N; ++n)
            for (int32_t j = h.node_off[n]; j < h.node_off[n + 1]; ++j) {
                const int32_t e = h.node_ent[j] >> 3;
                if (!h.state[e]) continue;
                const double w = h.V[e] / 8.0;
                for (int c = 0; c < 3; ++c) h.fext[3 * n + c] = h.fext[3 * n + c] + ld->body[c] * w;
                h.nflag[n] |= 8;
            }
    if (ld && ld->n_tfaces > 0) {
        if (!ld->tface || !ld->tface_t) {
            err = "cem_init_mesh: n_tfaces > 0 with NULL arrays";
            return CEM_EINVAL;
        }
        for (int64_t f = 0; f < ld->n_tfaces; ++f) {
            const int32_t *t = ld->tface + 3 * f;
            for (int i = 0; i < 3; ++i)
                if (t[i] < 0 || t[i] >= N) {
                    err = "traction face " + std::to_string(f) + ": node out of range";
                    return CEM_ETOPOLOGY;
                }
            const W3 x0 = {m->X[3 * (int64_t)t[0]], m->X[3 * (int64_t)t[0] + 1], m->X[3 * (int64_t)t[0] + 2]};
            const W3 x1 = {m->X[3 * (int64_t)t[1]], m->X[3 * (int64_t)t[1] + 1], m->X[3 * (int64_t)t[1] + 2]};
            const W3 x2 = {m->X[3 * (int64_t)t[2]], m->X[3 * (int64_t)t[2] + 1], m->X[3 * (int64_t)t[2] + 2]};
            const W3 cr = wcross(wsub(x1, x0), wsub(x2, x0));
            const double w = (0.5 * std::sqrt(wdot(cr, cr))) / 3.0;
            for (int i = 0; i < 3; ++i) {
                for (int c = 0; c < 3; ++c) h.fext[3 * (int64_t)t[i] + c] = h.fext[3 * (int64_t)t[i] + c] + ld->tface_t[3 * f + c] * w;
                h.nflag[t[i]] |= 8;
            }
        }
    }
    if (ld && ld->f_nodal)
        for (int64_t n = 0; n < N; ++n) {
            bool any = false;
            for (int c = 0; c < 3; ++c) {
                h.fext[3 * n + c] = h.fext[3 * n + c] + ld->f_nodal[3 * n + c];
                any = any || ld->f_nodal[3 * n + c] != 0.0;
            }
            if (any) h.nflag[n] |= 8;
        }
    if (ld && ld->n_vbc > 0) {
        if (!ld->vbc_node || !ld->vbc_mask || !ld->vbc_v0) {
            err = "cem_init_mesh: n_vbc > 0 with NULL arrays";
            return CEM_EINVAL;
        }
        for (int64_t b = 0; b < ld->n_vbc; ++b) {
            const int32_t n = ld->vbc_node[b];
            if (n < 0 || n >= N) {
                err = "prescribed-velocity node out of range";
                return CEM_ETOPOLOGY;
            }
            h.nflag[n] |= ld->vbc_mask[b] & 7;
            for (int c = 0; c < 3; ++c)
                if (ld->vbc_mask[b] >> c & 1) h.dir_v0[3 * (int64_t)n + c] = ld->vbc_v0[3 * b + c];
        }
        h.any_dirichlet = true;
        h.t0 = ld->vbc_t0;
    }
    // ---------------------------------------------------------------- time step (R25)
    double dt = o ? o->dt : 0.0;
    if (!(dt > 0)) {
        const double cd = std::sqrt(h.l2m / h.rho);
        double hmin = INFINITY;
        for (int64_t e = 0; e < E; ++e) {
            if (!h.state[e]) continue;
            double amax = 0.0;
            for (int f = 0; f < 6; ++f) {
                W3 x[4];
                for (int q = 0; q < 4; ++q) {
                    const int64_t n = h.hex[8 * e + kFace[f][q]];
                    x[q] = {m->X[3 * n], m->X[3 * n + 1], m->X[3 * n + 2]};
                }
                const W3 cr = wcross(wsub(x[2], x[0]), wsub(x[3], x[1]));
                const double A = 0.5 * std::sqrt(wdot(cr, cr));
                if (A > amax) amax = A;
            }
            const double he = h.V[e] / amax;
            if (he < hmin) hmin = he;
        }
        if (!std::isfinite(hmin)) {
            err = "no active hex to derive dt from";
            return CEM_EINVAL;
        }
        dt = (cfl * hmin) / cd;
    }
    h.dt = dt;
    // node -> force-slot ELL: incidence (e, a) owns slot 8e + a for the hex's force (the hexes' slots are
    // contiguous: 192 B per hex, written whole by stage C) and slots 8E + 3 (8e + a) + i for remainder
    // tet i (zero while unused).  Row of a node with k incidences: its k hex slots in
    // ascending e (the walk of hex_node_mass), then the 3k remainder slots, then the zero slot 32E.
    // The nodal sum is exact (R27), so its order is free; for a node of no remainder prism (hnrem == 0)
    // stage D reads only the first wn0 entries (every hex slot; any further entry still zero).
    int mx = 1;
    for (int64_t n = 0; n < N; ++n) mx = std::max(mx, h.node_off[n + 1] - h.node_off[n]);
    h.wn = (4 * mx + 7) / 8 * 8;
    h.wn0 = (mx + 7) / 8 * 8;
    h.zslot = (int32_t)(32 * E);
    h.nodeE.assign((size_t)N * h.wn, h.zslot);
    for (int64_t n = 0; n < N; ++n) {
        const int32_t j0 = h.node_off[n], k = h.node_off[n + 1] - j0;
        int32_t *row = h.nodeE.data() + (size_t)n * h.wn;
        for (int32_t j = 0; j < k; ++j) {
            row[j] = h.node_ent[j0 + j];
            for (int i = 0; i < 3; ++i) row[k + 3 * j + i] = (int32_t)(8 * E) + 3 * h.node_ent[j0 + j] + i;
        }
    }
    return CEM_OK;
}

}  // namespace cem
