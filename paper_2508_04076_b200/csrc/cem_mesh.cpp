// cem_mesh.cpp -- host preprocessing of libcem.so: validation, ES-FEM topology, geometry,
// lumped mass, traction force, time step.  Compiled with
// -ffp-contract=off so every expression rounds exactly as written (DESIGN.md
// "Association order"); OpenMP only over independent outputs.
#include <parallel/algorithm>
#include <algorithm>
#include <cmath>
#include <cstring>
#include <numeric>

#include "cem_internal.h"

namespace cem {

namespace {

const int kEdgeP[6] = {0, 0, 0, 1, 1, 2};
const int kEdgeQ[6] = {1, 2, 3, 2, 3, 3};
const int kFaceNodes[4][3] = {{1, 2, 3}, {0, 2, 3}, {0, 1, 3}, {0, 1, 2}};

struct V3 {
    double x, y, z;
};
inline V3 sub(V3 a, V3 b) { return {a.x - b.x, a.y - b.y, a.z - b.z}; }
inline double dot(V3 a, V3 b) { return (a.x * b.x + a.y * b.y) + a.z * b.z; }
inline V3 cross(V3 a, V3 b) { return {a.y * b.z - a.z * b.y, a.z * b.x - a.x * b.z, a.x * b.y - a.y * b.x}; }
inline V3 node(const double *X, int64_t n) { return {X[3 * n], X[3 * n + 1], X[3 * n + 2]}; }

// (lo << 32 | hi, 6e + l) pairs sorted by key then by tet-edge index
void edge_keys(const cem_mesh_in *m, std::vector<std::pair<uint64_t, int64_t>> &k) {
    const int64_t E = m->n_tets;
    k.resize(6 * E);
#pragma omp parallel for schedule(static)
    for (int64_t e = 0; e < E; ++e)
        for (int l = 0; l < 6; ++l) {
            uint64_t i = (uint32_t)m->tets[4 * e + kEdgeP[l]], j = (uint32_t)m->tets[4 * e + kEdgeQ[l]];
            uint64_t lo = std::min(i, j), hi = std::max(i, j);
            k[6 * e + l] = {lo << 32 | hi, 6 * e + l};
        }
    __gnu_parallel::sort(k.begin(), k.end());  // keys are unique pairs: the order is total
}

}  // namespace

cem_status count_edges(const cem_mesh_in *m, int64_t *S, std::string &err) {
    if (!m || !m->tets || m->n_tets <= 0) {
        err = "mesh has no tets";
        return CEM_EINVAL;
    }
    std::vector<std::pair<uint64_t, int64_t>> k;
    edge_keys(m, k);
    int64_t s = 0;
    for (size_t i = 0; i < k.size(); ++i)
        if (i == 0 || k[i].first != k[i - 1].first) ++s;
    *S = s;
    return CEM_OK;
}

// dt = cfl * min_{active e} (3 V_e / max face area_e) / c_d, c_d = sqrt((lam + 2 mu)/rho)
cem_status cfl_dt(int64_t N, const double *X, int64_t E, const int32_t *tets, const uint8_t *state, const double *V,
                  double l2m, double rho, double cfl, double *dt_out, std::string &err) {
    (void)N;
    const double cd = std::sqrt(l2m / rho);
    double altmin = INFINITY;
    for (int64_t e = 0; e < E; ++e) {
        if (!state[e]) continue;
        double amax = 0.0;
        for (int f = 0; f < 4; ++f) {
            const int32_t *t = tets + 4 * e;
            V3 x0 = node(X, t[kFaceNodes[f][0]]);
            V3 cr = cross(sub(node(X, t[kFaceNodes[f][1]]), x0), sub(node(X, t[kFaceNodes[f][2]]), x0));
            double A = 0.5 * std::sqrt(dot(cr, cr));
            if (A > amax) amax = A;
        }
        double alt = 3.0 * V[e] / amax;
        if (alt < altmin) altmin = alt;
    }
    if (!std::isfinite(altmin)) {
        err = "no active tet to derive dt from";
        return CEM_EINVAL;
    }
    *dt_out = (cfl * altmin) / cd;
    return CEM_OK;
}

// the same rule on a mesh given only by arrays (global dt of a partitioned run)
cem_status global_cfl_dt(const cem_mesh_in *m, const cem_material *mat, double cfl, double *dt, std::string &err) {
    const int64_t E = m->n_tets;
    std::vector<double> V(E);
    std::vector<uint8_t> st(E);
    for (int64_t e = 0; e < E; ++e) {
        const int32_t *t = m->tets + 4 * e;
        V3 x0 = node(m->X, t[0]);
        V3 d1 = sub(node(m->X, t[1]), x0), d2 = sub(node(m->X, t[2]), x0), d3 = sub(node(m->X, t[3]), x0);
        V[e] = dot(d1, cross(d2, d3)) / 6.0;
        st[e] = m->tet_state ? (m->tet_state[e] != 0) : 1;
    }
    const double lam = mat->E * mat->nu / ((1.0 + mat->nu) * (1.0 - 2.0 * mat->nu));
    const double mu = mat->E / (2.0 * (1.0 + mat->nu));
    return cfl_dt(m->n_nodes, m->X, E, m->tets, st.data(), V.data(), lam + 2.0 * mu, mat->rho, cfl, dt, err);
}

cem_status build_host_mesh(const cem_mesh_in *m, const cem_material *mat, const cem_load_in *ld,
                           const cem_opts *o, HostMesh &h, std::string &err) {
    if (!m || !mat || !m->X || !m->tets || m->n_nodes <= 0 || m->n_tets <= 0) {
        err = "cem_init_mesh: empty mesh or NULL array";
        return CEM_EINVAL;
    }
    if (!(mat->E > 0) || !(mat->nu > -1.0 && mat->nu < 0.5) || !(mat->rho > 0) || !(mat->Gc >= 0)) {
        err = "cem_init_mesh: material needs E > 0, -1 < nu < 0.5, rho > 0, Gc >= 0";
        return CEM_EINVAL;
    }
    const double gamma = o && o->gamma > 0 ? o->gamma : 0.5;
    const double cfl = o && o->cfl > 0 ? o->cfl : 0.5;
    if (gamma > 1.0) {
        err = "cem_init_mesh: gamma must be in (0, 1]";
        return CEM_EINVAL;
    }
    const int64_t N = m->n_nodes, E = m->n_tets;
    // index ranges of the device layout: 32-bit element offsets of 12 E force-slot doubles
    // (4 slots x 3 components per tet) and of the 6-E edge incidences (checked before any array
    // is read)
    if (E > ((int64_t)1 << 32) / 12 - 64 || N >= ((int64_t)1 << 31)) {
        err = "mesh too large for one context (E must be < 357M tets; partition it over ranks)";
        return CEM_EINVAL;
    }
    h.N = N;
    h.E = E;
    h.X.assign(m->X, m->X + 3 * N);
    h.tet.assign(m->tets, m->tets + 4 * E);
    h.state.resize(E);
    h.gc.resize(E);
    for (int64_t e = 0; e < E; ++e) {
        h.state[e] = m->tet_state ? (m->tet_state[e] != 0) : 1;
        h.gc[e] = m->tet_gc ? m->tet_gc[e] : mat->Gc;
    }
    PhaseClock clk;
    // ---------------------------------------------------------------- validation
    for (int64_t e = 0; e < E; ++e) {
        const int32_t *t = m->tets + 4 * e;
        for (int a = 0; a < 4; ++a) {
            if (t[a] < 0 || t[a] >= N) {
                err = "tet " + std::to_string(e) + ": node index out of range";
                return CEM_ETOPOLOGY;
            }
            for (int b = 0; b < a; ++b)
                if (t[a] == t[b]) {
                    err = "tet " + std::to_string(e) + ": repeated node";
                    return CEM_ETOPOLOGY;
                }
        }
    }
    double lo[3] = {INFINITY, INFINITY, INFINITY}, hi[3] = {-INFINITY, -INFINITY, -INFINITY};
    for (int64_t n = 0; n < N; ++n)
        for (int c = 0; c < 3; ++c) {
            double x = m->X[3 * n + c];
            if (!std::isfinite(x)) {
                err = "node " + std::to_string(n) + ": non-finite coordinate";
                return CEM_EINVAL;
            }
            lo[c] = std::min(lo[c], x);
            hi[c] = std::max(hi[c], x);
        }
    const double ext = std::max({hi[0] - lo[0], hi[1] - lo[1], hi[2] - lo[2]});
    const double vtol = 1e-14 * ext * ext * ext;
    clk.mark("mesh: validation");
    // ---------------------------------------------------------------- geometry
    // det = d1.(d2 x d3), V = det/6, inv = 1/det, gradN1 = (d2xd3) inv, gradN2 = (d3xd1) inv,
    // gradN3 = (d1xd2) inv, gradN0 = -((gradN1 + gradN2) + gradN3)
    h.V.assign(E, 0.0);
    h.grad.resize(12 * E);  // (written for every valid tet; an invalid one fails the init)
    int64_t bad_neg = -1, bad_deg = -1;
#pragma omp parallel for schedule(static)
    for (int64_t e = 0; e < E; ++e) {
        const int32_t *t = m->tets + 4 * e;
        V3 x0 = node(m->X, t[0]);
        V3 d1 = sub(node(m->X, t[1]), x0), d2 = sub(node(m->X, t[2]), x0), d3 = sub(node(m->X, t[3]), x0);
        V3 c23 = cross(d2, d3), c31 = cross(d3, d1), c12 = cross(d1, d2);
        double det = dot(d1, c23);
        double V = det / 6.0;
        double *g = h.grad.data() + 12 * e;
        if (det < 0) {
#pragma omp critical
            bad_neg = bad_neg < 0 ? e : std::min(bad_neg, e);
            continue;
        }
        if (V < vtol || V == 0.0) {
#pragma omp critical
            bad_deg = bad_deg < 0 ? e : std::min(bad_deg, e);
            continue;
        }
        double inv = 1.0 / det;
        h.V[e] = V;
        double gr[4][3];
        const double cc[3][3] = {{c23.x, c23.y, c23.z}, {c31.x, c31.y, c31.z}, {c12.x, c12.y, c12.z}};
        for (int a = 1; a < 4; ++a)
            for (int c = 0; c < 3; ++c) gr[a][c] = cc[a - 1][c] * inv;
        for (int c = 0; c < 3; ++c) gr[0][c] = -((gr[1][c] + gr[2][c]) + gr[3][c]);
        for (int a = 0; a < 4; ++a)
            for (int c = 0; c < 3; ++c) g[3 * a + c] = gr[a][c];
    }
    if (bad_neg >= 0) {
        err = "tet " + std::to_string(bad_neg) + ": negative orientation";
        return CEM_ENEGVOL;
    }
    if (bad_deg >= 0) {
        err = "tet " + std::to_string(bad_deg) + ": degenerate (|V| < 1e-14 bbox^3)";
        return CEM_EDEGENERATE;
    }
    clk.mark("mesh: geometry");
    // ---------------------------------------------------------------- duplicate tets
    {
        std::vector<std::pair<uint64_t, uint64_t>> tk(E);
#pragma omp parallel for schedule(static)
        for (int64_t e = 0; e < E; ++e) {
            int32_t v[4];
            std::memcpy(v, m->tets + 4 * e, sizeof v);
            std::sort(v, v + 4);
            tk[e] = {((uint64_t)(uint32_t)v[0] << 32) | (uint32_t)v[1], ((uint64_t)(uint32_t)v[2] << 32) | (uint32_t)v[3]};
        }
        __gnu_parallel::sort(tk.begin(), tk.end());
        for (int64_t e = 1; e < E; ++e)
            if (tk[e] == tk[e - 1]) {
                err = "duplicate tets (same node set)";
                return CEM_ETOPOLOGY;
            }
    }
    clk.mark("mesh: duplicate tets");
    // ---------------------------------------------------------------- edges (ES-FEM smoothing domains)
    // The unique (min, max) node pairs in lexicographic order, each with its incident tets in
    // ascending id -- the order of one global sort of the (lo, hi, 6e + l) keys, built as buckets
    // by lo (counting pass + scatter) each sorted by (hi, 6e + l): O(6E) plus small sorts, parallel.
    {
        const int64_t NE = 6 * E;
        std::vector<int32_t> boff(N + 1, 0);
#pragma omp parallel for schedule(static)
        for (int64_t e = 0; e < E; ++e)
            for (int l = 0; l < 6; ++l) {
                const int32_t i = m->tets[4 * e + kEdgeP[l]], j = m->tets[4 * e + kEdgeQ[l]];
                __atomic_fetch_add(&boff[std::min(i, j) + 1], 1, __ATOMIC_RELAXED);
            }
        for (int64_t n = 0; n < N; ++n) boff[n + 1] += boff[n];
        std::vector<uint64_t> item(NE);  // hi << 32 | (6e + l)   (6E < 2^32: cem_init_mesh's size limit)
        {
            std::vector<int32_t> fill(boff.begin(), boff.end() - 1);
#pragma omp parallel for schedule(static)
            for (int64_t e = 0; e < E; ++e)
                for (int l = 0; l < 6; ++l) {
                    const int32_t i = m->tets[4 * e + kEdgeP[l]], j = m->tets[4 * e + kEdgeQ[l]];
                    const int32_t pos = __atomic_fetch_add(&fill[std::min(i, j)], 1, __ATOMIC_RELAXED);
                    item[pos] = (uint64_t)(uint32_t)std::max(i, j) << 32 | (uint64_t)(6 * e + l);
                }
        }
        std::vector<int64_t> ecnt(N + 1, 0);  // distinct edges per bucket -> first edge id of a bucket
#pragma omp parallel for schedule(dynamic, 1024)
        for (int64_t n = 0; n < N; ++n) {
            std::sort(item.begin() + boff[n], item.begin() + boff[n + 1]);
            int64_t c = 0;
            for (int32_t i = boff[n]; i < boff[n + 1]; ++i)
                if (i == boff[n] || (item[i] >> 32) != (item[i - 1] >> 32)) ++c;
            ecnt[n + 1] = c;
        }
        for (int64_t n = 0; n < N; ++n) ecnt[n + 1] += ecnt[n];
        const int64_t S = ecnt[N];
        h.S = S;
        h.edge_nodes.resize(2 * S);
        h.edge_off.assign(S + 1, 0);
        h.edge_inc.resize(NE);
        h.elem_edge.resize(NE);
#pragma omp parallel for schedule(dynamic, 1024)
        for (int64_t n = 0; n < N; ++n) {
            int64_t s = ecnt[n] - 1;
            for (int32_t i = boff[n]; i < boff[n + 1]; ++i) {
                const uint32_t hi = (uint32_t)(item[i] >> 32), te = (uint32_t)item[i];
                if (i == boff[n] || hi != (uint32_t)(item[i - 1] >> 32)) {
                    ++s;
                    h.edge_nodes[2 * s] = (int32_t)n;
                    h.edge_nodes[2 * s + 1] = (int32_t)hi;
                    h.edge_off[s] = i;
                }
                h.edge_inc[i] = (int32_t)(te / 6);  // ascending tet id within an edge
                h.elem_edge[te] = (int32_t)s;
            }
        }
        h.edge_off[S] = (int32_t)NE;
    }
    clk.mark("mesh: edges");
    // ---------------------------------------------------------------- node incidence (ascending e)
    h.node_off.assign(N + 1, 0);
    for (int64_t i = 0; i < 4 * E; ++i) h.node_off[m->tets[i] + 1]++;
    for (int64_t n = 0; n < N; ++n) h.node_off[n + 1] += h.node_off[n];
    h.node_ent.resize(4 * E);
    {
        std::vector<int32_t> fill(h.node_off.begin(), h.node_off.end() - 1);
        for (int64_t e = 0; e < E; ++e)
            for (int a = 0; a < 4; ++a) h.node_ent[fill[m->tets[4 * e + a]]++] = (int32_t)(4 * e + a);
    }
    // ---------------------------------------------------------------- material
    h.rho = mat->rho;
    h.lam = mat->E * mat->nu / ((1.0 + mat->nu) * (1.0 - 2.0 * mat->nu));
    h.mu = mat->E / (2.0 * (1.0 + mat->nu));
    h.l2m = h.lam + 2.0 * h.mu;
    h.gamma = gamma;
    // ---------------------------------------------------------------- lumped mass: sum_{active e} (rho V_e)/4
    h.mass.assign(N, 0.0);
#pragma omp parallel for schedule(static)
    for (int64_t n = 0; n < N; ++n) {
        double acc = 0.0;
        for (int32_t j = h.node_off[n]; j < h.node_off[n + 1]; ++j) {
            int32_t e = h.node_ent[j] >> 2;
            if (!h.state[e]) continue;
            acc = acc + (h.rho * h.V[e]) / 4.0;
        }
        h.mass[n] = acc;
    }
    // ---------------------------------------------------------------- external force
    // body force b (V_e/4) over the active incident tets in ascending tet id, then the traction
    // triangles f_k += t (A/3) in the given order, then the nodal point forces (include/cem.h)
    h.fext.assign(3 * N, 0.0);
    h.nflag.assign(N, 0);
    h.dir_v0.assign(3 * N, 0.0);
    if (ld && (ld->body[0] != 0.0 || ld->body[1] != 0.0 || ld->body[2] != 0.0)) {
        if (!std::isfinite(ld->body[0]) || !std::isfinite(ld->body[1]) || !std::isfinite(ld->body[2])) {
            err = "cem_init_mesh: non-finite body force";
            return CEM_EINVAL;
        }
#pragma omp parallel for schedule(static)
        for (int64_t n = 0; n < N; ++n) {
            bool any = false;
            for (int32_t j = h.node_off[n]; j < h.node_off[n + 1]; ++j) {
                const int32_t e = h.node_ent[j] >> 2;
                if (!h.state[e]) continue;
                const double w = h.V[e] / 4.0;
                for (int c = 0; c < 3; ++c) h.fext[3 * n + c] = h.fext[3 * n + c] + ld->body[c] * w;
                any = true;
            }
            if (any) h.nflag[n] |= 8;
        }
    }
    if (ld && ld->n_tfaces > 0) {
        if (!ld->tface || !ld->tface_t) {
            err = "cem_init_mesh: n_tfaces > 0 with NULL arrays";
            return CEM_EINVAL;
        }
        for (int64_t f = 0; f < ld->n_tfaces; ++f) {
            const int32_t *tri = ld->tface + 3 * f;
            for (int i = 0; i < 3; ++i)
                if (tri[i] < 0 || tri[i] >= N) {
                    err = "traction face " + std::to_string(f) + ": node out of range";
                    return CEM_ETOPOLOGY;
                }
            V3 x0 = node(m->X, tri[0]);
            V3 cr = cross(sub(node(m->X, tri[1]), x0), sub(node(m->X, tri[2]), x0));
            double A = 0.5 * std::sqrt(dot(cr, cr));
            double w = A / 3.0;
            for (int i = 0; i < 3; ++i) {
                for (int c = 0; c < 3; ++c) h.fext[3 * (int64_t)tri[i] + c] = h.fext[3 * (int64_t)tri[i] + c] + ld->tface_t[3 * f + c] * w;
                h.nflag[tri[i]] |= 8;
            }
        }
    }
    if (ld && ld->f_nodal) {
        for (int64_t n = 0; n < N; ++n) {
            bool any = false;
            for (int c = 0; c < 3; ++c) {
                const double f = ld->f_nodal[3 * n + c];
                if (!std::isfinite(f)) {
                    err = "cem_init_mesh: non-finite f_nodal";
                    return CEM_EINVAL;
                }
                h.fext[3 * n + c] = h.fext[3 * n + c] + f;
                any = any || f != 0.0;
            }
            if (any) h.nflag[n] |= 8;
        }
    }
    if (ld && ld->n_vbc > 0) {
        if (!ld->vbc_node || !ld->vbc_mask || !ld->vbc_v0) {
            err = "cem_init_mesh: n_vbc > 0 with NULL arrays";
            return CEM_EINVAL;
        }
        for (int64_t b = 0; b < ld->n_vbc; ++b) {
            int32_t k = ld->vbc_node[b];
            if (k < 0 || k >= N) {
                err = "prescribed-velocity node out of range";
                return CEM_ETOPOLOGY;
            }
            h.nflag[k] |= ld->vbc_mask[b] & 7;
            for (int c = 0; c < 3; ++c)
                if (ld->vbc_mask[b] >> c & 1) h.dir_v0[3 * (int64_t)k + c] = ld->vbc_v0[3 * b + c];
        }
        h.any_dirichlet = true;
        h.t0 = ld->vbc_t0;
    }
    clk.mark("mesh: incidence/mass/loads");
    // ---------------------------------------------------------------- time step (R12)
    double dt = o ? o->dt : 0.0;
    if (!(dt > 0)) {
        cem_status st = cfl_dt(m->n_nodes, m->X, m->n_tets, m->tets, h.state.data(), h.V.data(), h.l2m, h.rho, cfl, &dt, err);
        if (st) return st;
    }
    h.dt = dt;
    return CEM_OK;
}

}  // namespace cem
