// cem_plan.cpp -- storage numbering, block decomposition and the wavefront schedule of the
// persistent step kernel ("Persistent wavefront").
//
// Storage order: tets sorted by (slab index of the centroid along the longest bounding-box
// axis, original id) with slab width (6 mean V)^(1/3) ~ one element layer; nodes and edges
// numbered by first appearance in that tet order.  A consumer block then depends only on a
// narrow range of producer blocks (about one element layer), which keeps every
// intermediate (tau, sigma, f_e) L2-resident between its producer and consumer.
// Summation lists (edge -> tets, node -> tets) stay in ORIGINAL tet-id order.
#include <algorithm>
#include <cmath>
#include <numeric>

#include "cem_internal.h"

namespace cem {

void build_plan(const HostMesh &h, int blk, int resident_ctas, Plan &p) {
    const int64_t N = h.N, E = h.E, S = h.S;
    p.blk = blk;
    // ---------------------------------------------------------------- sweep axis + slabs
    double lo[3] = {INFINITY, INFINITY, INFINITY}, hi[3] = {-INFINITY, -INFINITY, -INFINITY};
    for (int64_t n = 0; n < N; ++n)
        for (int c = 0; c < 3; ++c) {
            lo[c] = std::min(lo[c], h.X[3 * n + c]);
            hi[c] = std::max(hi[c], h.X[3 * n + c]);
        }
    int ax = 0;
    for (int c = 1; c < 3; ++c)
        if (hi[c] - lo[c] > hi[ax] - lo[ax]) ax = c;
    double vsum = 0.0;
    for (int64_t e = 0; e < E; ++e) vsum += h.V[e];
    const double hb = std::cbrt(6.0 * vsum / (double)E);
    std::vector<int64_t> key(E);
    for (int64_t e = 0; e < E; ++e) {
        double c = 0.0;
        for (int a = 0; a < 4; ++a) c += h.X[3 * (int64_t)h.tet[4 * e + a] + ax];
        c *= 0.25;
        key[e] = (int64_t)std::floor((c - lo[ax]) / hb);
    }
    p.tet_new2old.resize(E);
    std::iota(p.tet_new2old.begin(), p.tet_new2old.end(), 0);
    std::stable_sort(p.tet_new2old.begin(), p.tet_new2old.end(),
                     [&](int32_t x, int32_t y) { return key[x] < key[y]; });
    p.tet_old2new.assign(E, -1);
    for (int64_t e = 0; e < E; ++e) p.tet_old2new[p.tet_new2old[e]] = (int32_t)e;
    // nodes and edges by first appearance
    p.node_old2new.assign(N, -1);
    p.node_new2old.clear();
    p.node_new2old.reserve(N);
    std::vector<int32_t> edge_old2new(S, -1);
    p.edge_new2old.clear();
    p.edge_new2old.reserve(S);
    for (int64_t en = 0; en < E; ++en) {
        const int64_t eo = p.tet_new2old[en];
        for (int a = 0; a < 4; ++a) {
            int32_t k = h.tet[4 * eo + a];
            if (p.node_old2new[k] < 0) {
                p.node_old2new[k] = (int32_t)p.node_new2old.size();
                p.node_new2old.push_back(k);
            }
        }
        for (int l = 0; l < 6; ++l) {
            int32_t s = h.elem_edge[6 * eo + l];
            if (edge_old2new[s] < 0) {
                edge_old2new[s] = (int32_t)p.edge_new2old.size();
                p.edge_new2old.push_back(s);
            }
        }
    }
    for (int64_t k = 0; k < N; ++k)  // nodes referenced by no tet go last
        if (p.node_old2new[k] < 0) {
            p.node_old2new[k] = (int32_t)p.node_new2old.size();
            p.node_new2old.push_back((int32_t)k);
        }
    // ---------------------------------------------------------------- storage-order tables
    p.conn.resize(4 * E);
    p.geoV.resize(E);
    p.geoC.resize(E);
    p.geoG.resize(9 * E);
    p.eedge.resize(6 * E);
    p.state.resize(E);
    p.gc.resize(E);
    for (int64_t en = 0; en < E; ++en) {
        const int64_t eo = p.tet_new2old[en];
        for (int a = 0; a < 4; ++a) p.conn[4 * en + a] = p.node_old2new[h.tet[4 * eo + a]];
        p.geoV[en] = h.V[eo];
        p.geoC[en] = h.V[eo] / 6.0;
        for (int a = 1; a < 4; ++a)
            for (int c = 0; c < 3; ++c) p.geoG[(int64_t)(3 * (a - 1) + c) * E + en] = h.grad[12 * eo + 3 * a + c];
        for (int l = 0; l < 6; ++l) p.eedge[(int64_t)l * E + en] = edge_old2new[h.elem_edge[6 * eo + l]];
        p.state[en] = h.state[eo];
        p.gc[en] = h.gc[eo];
    }
    p.edge_off.assign(S + 1, 0);
    p.edge_inc.resize(h.edge_inc.size());
    for (int64_t sn = 0, j = 0; sn < S; ++sn) {
        const int32_t so = p.edge_new2old[sn];
        p.edge_off[sn] = (int32_t)j;
        for (int32_t i = h.edge_off[so]; i < h.edge_off[so + 1]; ++i) p.edge_inc[j++] = p.tet_old2new[h.edge_inc[i]];
        p.edge_off[sn + 1] = (int32_t)j;
    }
    p.node_off.assign(N + 1, 0);
    p.node_ent.resize(h.node_ent.size());
    for (int64_t kn = 0, j = 0; kn < N; ++kn) {
        const int32_t ko = p.node_new2old[kn];
        p.node_off[kn] = (int32_t)j;
        for (int32_t i = h.node_off[ko]; i < h.node_off[ko + 1]; ++i) {
            const int32_t ent = h.node_ent[i];
            p.node_ent[j++] = (p.tet_old2new[ent >> 2] << 2) | (ent & 3);
        }
        p.node_off[kn + 1] = (int32_t)j;
    }
    // ---------------------------------------------------------------- blocks and dependencies
    const int64_t cnt[ST_COUNT] = {E, S, E, N};
    p.maxblk = 0;
    for (int g = 0; g < ST_COUNT; ++g) {
        p.nblk[g] = (int)((cnt[g] + blk - 1) / blk);
        p.maxblk = std::max(p.maxblk, p.nblk[g]);
    }
    p.dep.assign((size_t)ST_COUNT * p.maxblk * 2, 0);
    auto setdep = [&](int g, int b, int lo_, int hi_) {
        p.dep[((size_t)g * p.maxblk + b) * 2] = lo_;
        p.dep[((size_t)g * p.maxblk + b) * 2 + 1] = hi_;
    };
    // A-block: D-blocks (previous step) of the nodes of its tets
    for (int b = 0; b < p.nblk[ST_A]; ++b) {
        int l = INT32_MAX, u = -1;
        for (int64_t e = (int64_t)b * blk; e < std::min<int64_t>(E, (int64_t)(b + 1) * blk); ++e)
            for (int a = 0; a < 4; ++a) {
                int nb = p.conn[4 * e + a] / blk;
                l = std::min(l, nb);
                u = std::max(u, nb);
            }
        setdep(ST_A, b, l, u);
    }
    // B-block: A-blocks of the tets incident to its edges
    for (int b = 0; b < p.nblk[ST_B]; ++b) {
        int l = INT32_MAX, u = -1;
        for (int64_t s = (int64_t)b * blk; s < std::min<int64_t>(S, (int64_t)(b + 1) * blk); ++s)
            for (int32_t j = p.edge_off[s]; j < p.edge_off[s + 1]; ++j) {
                int tb = p.edge_inc[j] / blk;
                l = std::min(l, tb);
                u = std::max(u, tb);
            }
        setdep(ST_B, b, l, u);
    }
    // C-block: B-blocks of the edges of its tets
    for (int b = 0; b < p.nblk[ST_C]; ++b) {
        int l = INT32_MAX, u = -1;
        for (int64_t e = (int64_t)b * blk; e < std::min<int64_t>(E, (int64_t)(b + 1) * blk); ++e)
            for (int q = 0; q < 6; ++q) {
                int sb = p.eedge[(int64_t)q * E + e] / blk;
                l = std::min(l, sb);
                u = std::max(u, sb);
            }
        setdep(ST_C, b, l, u);
    }
    // D-block: C-blocks of the tets incident to its nodes (isolated nodes: none)
    for (int b = 0; b < p.nblk[ST_D]; ++b) {
        int l = INT32_MAX, u = -1;
        for (int64_t k = (int64_t)b * blk; k < std::min<int64_t>(N, (int64_t)(b + 1) * blk); ++k)
            for (int32_t j = p.node_off[k]; j < p.node_off[k + 1]; ++j) {
                int tb = (p.node_ent[j] >> 2) / blk;
                l = std::min(l, tb);
                u = std::max(u, tb);
            }
        if (u < 0) l = 0, u = -1;  // empty range
        setdep(ST_D, b, l, u);
    }
    // ---------------------------------------------------------------- wavefront schedule
    // virtual time: vt(A, b) = b / nA; a consumer sits delta after its latest producer,
    // delta = (resident CTAs) / (items per step), so by the time a CTA dequeues it its
    // producers have normally completed.  Sorted by vt this is a topological order.
    const int P = p.nblk[0] + p.nblk[1] + p.nblk[2] + p.nblk[3];
    const double delta = std::max(1.0, (double)resident_ctas) / (double)P;
    std::vector<double> vt[ST_COUNT];
    for (int g = 0; g < ST_COUNT; ++g) vt[g].assign(p.nblk[g], 0.0);
    for (int b = 0; b < p.nblk[ST_A]; ++b) vt[ST_A][b] = (double)b / (double)p.nblk[ST_A];
    for (int g = ST_B; g <= ST_D; ++g)
        for (int b = 0; b < p.nblk[g]; ++b) {
            const int l = p.dep[((size_t)g * p.maxblk + b) * 2], u = p.dep[((size_t)g * p.maxblk + b) * 2 + 1];
            double m = 0.0;
            for (int q = l; q <= u; ++q) m = std::max(m, vt[g - 1][q]);
            vt[g][b] = m + delta;
        }
    std::vector<std::pair<double, int32_t>> items;
    items.reserve(P);
    for (int g = 0; g < ST_COUNT; ++g)
        for (int b = 0; b < p.nblk[g]; ++b) items.push_back({vt[g][b], (g << 28) | b});
    std::stable_sort(items.begin(), items.end(), [](const std::pair<double, int32_t> &x, const std::pair<double, int32_t> &y) {
        return x.first < y.first || (x.first == y.first && (x.second >> 28) < (y.second >> 28));
    });
    p.sched.resize(P);
    for (int i = 0; i < P; ++i) p.sched[i] = items[i].second;
}

}  // namespace cem
