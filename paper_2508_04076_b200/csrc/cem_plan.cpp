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

void build_plan(const HostMesh &h, int blk, Plan &p, const uint8_t *tflag_orig) {
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
    // slabs of kSlab element layers along the sweep axis; inside a slab, recursive
    // coordinate bisection of the tet centroids down to leaves of <= blk/2 tets, leaves in
    // tree order -> every block of blk consecutive tets is a compact 3D patch
    const int kSlab = 4;
    std::vector<double> cen(3 * E);
    std::vector<int64_t> key(E);
    for (int64_t e = 0; e < E; ++e) {
        for (int c = 0; c < 3; ++c) {
            double x = 0.0;
            for (int a = 0; a < 4; ++a) x += h.X[3 * (int64_t)h.tet[4 * e + a] + c];
            cen[3 * e + c] = 0.25 * x;
        }
        key[e] = (int64_t)std::floor((cen[3 * e + ax] - lo[ax]) / (kSlab * hb));
    }
    p.tet_new2old.resize(E);
    std::iota(p.tet_new2old.begin(), p.tet_new2old.end(), 0);
    std::stable_sort(p.tet_new2old.begin(), p.tet_new2old.end(),
                     [&](int32_t x, int32_t y) { return key[x] < key[y]; });
    {
        const int64_t leaf = std::max(1, blk / 2);
        std::vector<std::pair<int64_t, int64_t>> stack;
        int64_t i0 = 0;
        while (i0 < E) {  // one slab at a time
            int64_t i1 = i0;
            while (i1 < E && key[p.tet_new2old[i1]] == key[p.tet_new2old[i0]]) ++i1;
            stack.push_back({i0, i1});
            while (!stack.empty()) {
                auto [a0, a1] = stack.back();
                stack.pop_back();
                if (a1 - a0 <= leaf) continue;
                double mn[3] = {INFINITY, INFINITY, INFINITY}, mx[3] = {-INFINITY, -INFINITY, -INFINITY};
                for (int64_t i = a0; i < a1; ++i)
                    for (int c = 0; c < 3; ++c) {
                        mn[c] = std::min(mn[c], cen[3 * (int64_t)p.tet_new2old[i] + c]);
                        mx[c] = std::max(mx[c], cen[3 * (int64_t)p.tet_new2old[i] + c]);
                    }
                int cx = 0;
                for (int c = 1; c < 3; ++c)
                    if (mx[c] - mn[c] > mx[cx] - mn[cx]) cx = c;
                const int64_t mid = a0 + (a1 - a0) / 2;
                std::nth_element(p.tet_new2old.begin() + a0, p.tet_new2old.begin() + mid, p.tet_new2old.begin() + a1,
                                 [&](int32_t x, int32_t y) {
                                     const double u = cen[3 * (int64_t)x + cx], v = cen[3 * (int64_t)y + cx];
                                     return u < v || (u == v && x < y);
                                 });
                stack.push_back({mid, a1});  // right half processed after the left half
                stack.push_back({a0, mid});
            }
            i0 = i1;
        }
    }
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
    p.tflag.resize(E);
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
        p.tflag[en] = tflag_orig ? tflag_orig[eo] : 3;
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
    // ---------------------------------------------------------------- gather lists
    {
        const int nbt = (int)((E + blk - 1) / blk), nbs = (int)((S + blk - 1) / blk);
        p.nl_off.assign(nbt + 1, 0);
        p.el_off.assign(nbt + 1, 0);
        p.nl.clear();
        p.el.clear();
        p.lconn.assign(4 * E, 0);
        p.ledge.assign(8 * E, 0);
        p.max_nl = p.max_el = p.max_tl = 0;
        std::vector<int32_t> tmp;
        for (int b = 0; b < nbt; ++b) {
            const int64_t e0 = (int64_t)b * blk, e1 = std::min<int64_t>(E, e0 + blk);
            tmp.assign(p.conn.begin() + 4 * e0, p.conn.begin() + 4 * e1);
            std::sort(tmp.begin(), tmp.end());
            tmp.erase(std::unique(tmp.begin(), tmp.end()), tmp.end());
            for (int64_t e = e0; e < e1; ++e)
                for (int a = 0; a < 4; ++a)
                    p.lconn[4 * e + a] = (uint16_t)(std::lower_bound(tmp.begin(), tmp.end(), p.conn[4 * e + a]) - tmp.begin());
            p.nl.insert(p.nl.end(), tmp.begin(), tmp.end());
            p.nl_off[b + 1] = (int32_t)p.nl.size();
            p.max_nl = std::max(p.max_nl, (int)tmp.size());
            tmp.clear();
            for (int64_t e = e0; e < e1; ++e)
                for (int l = 0; l < 6; ++l) tmp.push_back(p.eedge[(int64_t)l * E + e]);
            std::sort(tmp.begin(), tmp.end());
            tmp.erase(std::unique(tmp.begin(), tmp.end()), tmp.end());
            for (int64_t e = e0; e < e1; ++e)
                for (int l = 0; l < 6; ++l)
                    p.ledge[8 * e + l] =
                        (uint16_t)(std::lower_bound(tmp.begin(), tmp.end(), p.eedge[(int64_t)l * E + e]) - tmp.begin());
            p.el.insert(p.el.end(), tmp.begin(), tmp.end());
            p.el_off[b + 1] = (int32_t)p.el.size();
            p.max_el = std::max(p.max_el, (int)tmp.size());
        }
        p.tl_off.assign(nbs + 1, 0);
        p.tl.clear();
        p.inc_local.assign(p.edge_inc.size(), 0);
        for (int b = 0; b < nbs; ++b) {
            const int64_t s0 = (int64_t)b * blk, s1 = std::min<int64_t>(S, s0 + blk);
            tmp.assign(p.edge_inc.begin() + p.edge_off[s0], p.edge_inc.begin() + p.edge_off[s1]);
            std::sort(tmp.begin(), tmp.end());
            tmp.erase(std::unique(tmp.begin(), tmp.end()), tmp.end());
            for (int32_t j = p.edge_off[s0]; j < p.edge_off[s1]; ++j)
                p.inc_local[j] = (uint16_t)(std::lower_bound(tmp.begin(), tmp.end(), p.edge_inc[j]) - tmp.begin());
            p.tl.insert(p.tl.end(), tmp.begin(), tmp.end());
            p.tl_off[b + 1] = (int32_t)p.tl.size();
            p.max_tl = std::max(p.max_tl, (int)tmp.size());
        }
        // nodes of each edge block's tet list (the fused AB stage recomputes tau from them)
        p.nlb_off.assign(nbs + 1, 0);
        p.nlb.clear();
        p.tconn.assign(4 * p.tl.size(), 0);
        p.max_nlb = 0;
        std::vector<int32_t> nodes;
        for (int b = 0; b < nbs; ++b) {
            nodes.clear();
            for (int32_t i = p.tl_off[b]; i < p.tl_off[b + 1]; ++i)
                for (int a = 0; a < 4; ++a) nodes.push_back(p.conn[4 * (int64_t)p.tl[i] + a]);
            std::sort(nodes.begin(), nodes.end());
            nodes.erase(std::unique(nodes.begin(), nodes.end()), nodes.end());
            for (int32_t i = p.tl_off[b]; i < p.tl_off[b + 1]; ++i)
                for (int a = 0; a < 4; ++a)
                    p.tconn[4 * (int64_t)i + a] = (uint16_t)(std::lower_bound(nodes.begin(), nodes.end(),
                                                                               p.conn[4 * (int64_t)p.tl[i] + a]) - nodes.begin());
            p.nlb.insert(p.nlb.end(), nodes.begin(), nodes.end());
            p.nlb_off[b + 1] = (int32_t)p.nlb.size();
            p.max_nlb = std::max(p.max_nlb, (int)nodes.size());
        }
        // node-major force slots, interleaved per warp of 32 consecutive nodes so that the
        // lanes of stage D read 32 consecutive slots per incidence index j
        const int64_t ng = (N + 31) / 32;
        p.gbase.assign(ng + 1, 0);
        for (int64_t g = 0; g < ng; ++g) {
            int32_t mx = 0;
            for (int64_t k = 32 * g; k < std::min<int64_t>(N, 32 * g + 32); ++k) mx = std::max(mx, p.node_off[k + 1] - p.node_off[k]);
            p.gbase[g + 1] = p.gbase[g] + 32 * mx;
        }
        p.nslots = 4 * E;  // tet-major force records (node_ent (e<<2|a) indexes them directly)
        p.fpos.assign(4 * E, -1);
        for (int64_t k = 0; k < N; ++k)
            for (int32_t j = p.node_off[k]; j < p.node_off[k + 1]; ++j)
                p.fpos[4 * (int64_t)(p.node_ent[j] >> 2) + (p.node_ent[j] & 3)] =
                    p.gbase[k / 32] + 32 * (j - p.node_off[k]) + (int32_t)(k % 32);
    }
    // ---------------------------------------------------------------- instruction-lean layouts
    {
        const int64_t nt = (E + 31) / 32;
        p.geoT.assign(nt * 11 * 32, 0.0);
        for (int64_t e = 0; e < E; ++e) {
            double *g = p.geoT.data() + (e >> 5) * 352 + (e & 31);
            g[0] = p.geoV[e];
            g[32] = p.geoC[e];
            for (int c = 0; c < 9; ++c) g[32 * (2 + c)] = p.geoG[(int64_t)c * E + e];
        }
        int mx = 1;
        for (int64_t s = 0; s < S; ++s) mx = std::max(mx, p.edge_off[s + 1] - p.edge_off[s]);
        p.we = (mx + 7) / 8 * 8;
        p.we_max = mx;
        p.incE.assign((size_t)S * p.we, 0xFFFF);
        for (int64_t s = 0; s < S; ++s)
            for (int32_t j = p.edge_off[s]; j < p.edge_off[s + 1]; ++j) p.incE[(size_t)s * p.we + (j - p.edge_off[s])] = p.inc_local[j];
        mx = 1;
        for (int64_t k = 0; k < N; ++k) mx = std::max(mx, p.node_off[k + 1] - p.node_off[k]);
        p.wn = (mx + 7) / 8 * 8;
        p.zslot = (int32_t)(((E + 31) / 32) * 128);  // first slot past the last tile: kept zero
        p.nodeE.assign((size_t)N * p.wn, p.zslot);
        for (int64_t k = 0; k < N; ++k)
            for (int32_t j = p.node_off[k]; j < p.node_off[k + 1]; ++j) {
                const int64_t e = p.node_ent[j] >> 2, a = p.node_ent[j] & 3;
                p.nodeE[(size_t)k * p.wn + (j - p.node_off[k])] = (int32_t)((((e >> 5) * 4 + a) << 5) + (e & 31));
            }
    }
    // ---------------------------------------------------------------- blocks and dependencies
    const int64_t cnt[ST_COUNT] = {S, E, N};
    p.maxblk = 0;
    for (int g = 0; g < ST_COUNT; ++g) {
        p.nblk[g] = (int)((cnt[g] + blk - 1) / blk);
        p.maxblk = std::max(p.maxblk, p.nblk[g]);
    }
    // explicit producer-block lists per (stage, block)
    std::vector<std::vector<int32_t>> deps((size_t)ST_COUNT * p.maxblk);
    auto finish = [](std::vector<int32_t> &v) {
        std::sort(v.begin(), v.end());
        v.erase(std::unique(v.begin(), v.end()), v.end());
    };
    for (int b = 0; b < p.nblk[ST_AB]; ++b) {  // AB: D-blocks (previous step) of its tet list's nodes
        auto &v = deps[(size_t)ST_AB * p.maxblk + b];
        for (int32_t i = p.nlb_off[b]; i < p.nlb_off[b + 1]; ++i) v.push_back(p.nlb[i] / blk);
        finish(v);
    }
    for (int b = 0; b < p.nblk[ST_C]; ++b) {  // C: AB-blocks of its edge list
        auto &v = deps[(size_t)ST_C * p.maxblk + b];
        for (int32_t i = p.el_off[b]; i < p.el_off[b + 1]; ++i) v.push_back(p.el[i] / blk);
        finish(v);
    }
    for (int b = 0; b < p.nblk[ST_D]; ++b) {  // D: C-blocks of the tets of its nodes
        auto &v = deps[(size_t)ST_D * p.maxblk + b];
        for (int64_t k = (int64_t)b * blk; k < std::min<int64_t>(N, (int64_t)(b + 1) * blk); ++k)
            for (int32_t j = p.node_off[k]; j < p.node_off[k + 1]; ++j) v.push_back((p.node_ent[j] >> 2) / blk);
        finish(v);
    }
    p.ncons.assign((size_t)ST_COUNT * p.maxblk, 0);
    for (int g = ST_C; g <= ST_D; ++g)
        for (int b = 0; b < p.nblk[g]; ++b)
            for (int32_t pb : deps[(size_t)g * p.maxblk + b]) p.ncons[(size_t)(g - 1) * p.maxblk + pb]++;
    p.dep_off.assign((size_t)ST_COUNT * p.maxblk + 1, 0);
    p.dep.clear();
    for (size_t q = 0; q < deps.size(); ++q) {
        p.dep.insert(p.dep.end(), deps[q].begin(), deps[q].end());
        p.dep_off[q + 1] = (int32_t)p.dep.size();
    }
}

void build_schedule(Plan &p, int resident_ctas) {
    // ---------------------------------------------------------------- wavefront schedule
    // virtual time: vt(A, b) = b / nA; a consumer sits delta after its latest producer,
    // delta = (resident CTAs) / (items per step), so by the time a CTA dequeues it its
    // producers have normally completed.  Sorted by vt this is a topological order.
    int P = 0;
    for (int g = 0; g < ST_COUNT; ++g) P += p.nblk[g];
    const double delta = std::max(1.0, (double)resident_ctas) / (double)P;
    std::vector<double> vt[ST_COUNT];
    for (int g = 0; g < ST_COUNT; ++g) vt[g].assign(p.nblk[g], 0.0);
    for (int b = 0; b < p.nblk[ST_AB]; ++b) vt[ST_AB][b] = (double)b / (double)p.nblk[ST_AB];
    for (int g = ST_C; g <= ST_D; ++g)
        for (int b = 0; b < p.nblk[g]; ++b) {
            double m = 0.0;
            const size_t q = (size_t)g * p.maxblk + b;
            for (int32_t i = p.dep_off[q]; i < p.dep_off[q + 1]; ++i) m = std::max(m, vt[g - 1][p.dep[i]]);
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
