// cem_part.cpp -- domain decomposition for the multi-GPU step.
//
// Every rank builds the same plan from the same global mesh (deterministic, no communication):
//  * tets: recursive coordinate bisection of the centroids into P parts (longest extent,
//    split at the rank-proportional count, ties by tet id);
//  * a node is owned by the owner of its lowest-id incident tet (isolated nodes: rank 0);
//  * layer 1 of rank p: owned tets + every tet incident to an owned node (f_int of an owned
//    node is then complete); ghost tets: tets sharing an edge with a layer-1 tet (the ES-FEM
//    2-ring: sigma of every edge of a layer-1 tet is then complete);
//  * local tets / nodes are kept in ascending GLOBAL id, so every per-edge and per-node sum
//    runs in the same order as on one GPU: results are bitwise independent of P;
//  * the crack criterion runs on all layer-1 tets (identical inputs -> identical decisions on
//    every rank that holds the tet); only the owner records the split;
//  * per step, owners send the predicted displacement of their nodes to the ranks holding
//    them, and the state byte of their tets to the ranks holding them as ghosts.
#include <algorithm>
#include <cmath>
#include <numeric>

#include "cem_part.h"

namespace cem {

static const int kEP[6] = {0, 0, 0, 1, 1, 2};
static const int kEQ[6] = {1, 2, 3, 2, 3, 3};

static void rcb(const std::vector<double> &cen, std::vector<int32_t> &idx, int64_t lo, int64_t hi, int p0, int np,
                std::vector<int32_t> &part) {
    if (np == 1) {
        for (int64_t i = lo; i < hi; ++i) part[idx[i]] = p0;
        return;
    }
    double mn[3] = {INFINITY, INFINITY, INFINITY}, mx[3] = {-INFINITY, -INFINITY, -INFINITY};
    for (int64_t i = lo; i < hi; ++i)
        for (int c = 0; c < 3; ++c) {
            mn[c] = std::min(mn[c], cen[3 * (int64_t)idx[i] + c]);
            mx[c] = std::max(mx[c], cen[3 * (int64_t)idx[i] + c]);
        }
    int ax = 0;
    for (int c = 1; c < 3; ++c)
        if (mx[c] - mn[c] > mx[ax] - mn[ax]) ax = c;
    const int npl = np / 2;
    const int64_t mid = lo + (hi - lo) * npl / np;
    // (the comparator is a strict total order: the set below `mid` is unique, so a selection gives the
    // same parts as a full sort, in O(n) per level instead of O(n log n))
    std::nth_element(idx.begin() + lo, idx.begin() + mid, idx.begin() + hi, [&](int32_t a, int32_t b) {
        const double u = cen[3 * (int64_t)a + ax], v = cen[3 * (int64_t)b + ax];
        return u < v || (u == v && a < b);
    });
    rcb(cen, idx, lo, mid, p0, npl, part);
    rcb(cen, idx, mid, hi, p0 + npl, np - npl, part);
}

void build_partition(int64_t N, const double *X, int64_t E, const int32_t *tet, int P, PartGlobal &g) {
    g.P = P;
    std::vector<double> cen(3 * E);
    for (int64_t e = 0; e < E; ++e)
        for (int c = 0; c < 3; ++c) {
            double x = 0.0;
            for (int a = 0; a < 4; ++a) x += X[3 * (int64_t)tet[4 * e + a] + c];
            cen[3 * e + c] = 0.25 * x;
        }
    g.tet_owner.assign(E, 0);
    std::vector<int32_t> idx(E);
    std::iota(idx.begin(), idx.end(), 0);
    rcb(cen, idx, 0, E, 0, P, g.tet_owner);
    // node owner = owner of the lowest-id incident tet
    g.node_owner.assign(N, -1);
    for (int64_t e = 0; e < E; ++e)
        for (int a = 0; a < 4; ++a) {
            const int32_t k = tet[4 * e + a];
            if (g.node_owner[k] < 0) g.node_owner[k] = g.tet_owner[e];
        }
    for (int64_t k = 0; k < N; ++k)
        if (g.node_owner[k] < 0) g.node_owner[k] = 0;
    // node -> tets and edge -> tets incidence (global)
    g.node_off.assign(N + 1, 0);
    for (int64_t i = 0; i < 4 * E; ++i) g.node_off[tet[i] + 1]++;
    for (int64_t k = 0; k < N; ++k) g.node_off[k + 1] += g.node_off[k];
    g.node_tets.resize(4 * E);
    {
        std::vector<int32_t> fill(g.node_off.begin(), g.node_off.end() - 1);
        for (int64_t e = 0; e < E; ++e)
            for (int a = 0; a < 4; ++a) g.node_tets[fill[tet[4 * e + a]]++] = (int32_t)e;
    }
    std::vector<std::pair<uint64_t, int32_t>> keys(6 * E);
    for (int64_t e = 0; e < E; ++e)
        for (int l = 0; l < 6; ++l) {
            uint64_t i = (uint32_t)tet[4 * e + kEP[l]], j = (uint32_t)tet[4 * e + kEQ[l]];
            keys[6 * e + l] = {std::min(i, j) << 32 | std::max(i, j), (int32_t)e};
        }
    std::sort(keys.begin(), keys.end());
    g.tet_edge.assign(6 * E, 0);
    g.edge_off.clear();
    g.edge_tets.resize(6 * E);
    int64_t S = -1;
    for (size_t i = 0; i < keys.size(); ++i) {
        if (i == 0 || keys[i].first != keys[i - 1].first) {
            ++S;
            g.edge_off.push_back((int32_t)i);
        }
        g.edge_tets[i] = keys[i].second;
    }
    g.edge_off.push_back((int32_t)keys.size());
    // tet -> its 6 edge ids
    {
        std::vector<int32_t> cnt(E, 0);
        for (int64_t s = 0; s + 1 < (int64_t)g.edge_off.size(); ++s)
            for (int32_t j = g.edge_off[s]; j < g.edge_off[s + 1]; ++j) {
                const int32_t e = g.edge_tets[j];
                g.tet_edge[6 * (int64_t)e + cnt[e]++] = (int32_t)s;
            }
    }
    // per-rank local sets
    g.local_tets.assign(P, {});
    g.layer1.assign(P, {});
    g.local_nodes.assign(P, {});
    std::vector<uint8_t> mark(E);
    std::vector<uint8_t> nmark(N);
    for (int p = 0; p < P; ++p) {
        std::fill(mark.begin(), mark.end(), 0);
        for (int64_t k = 0; k < N; ++k)
            if (g.node_owner[k] == p)
                for (int32_t j = g.node_off[k]; j < g.node_off[k + 1]; ++j) mark[g.node_tets[j]] = 2;
        for (int64_t e = 0; e < E; ++e)
            if (g.tet_owner[e] == p) mark[e] = 2;
        for (int64_t e = 0; e < E; ++e)  // ghost ring: share an edge with a layer-1 tet
            if (mark[e] == 2)
                for (int l = 0; l < 6; ++l) {
                    const int32_t s = g.tet_edge[6 * e + l];
                    for (int32_t j = g.edge_off[s]; j < g.edge_off[s + 1]; ++j)
                        if (!mark[g.edge_tets[j]]) mark[g.edge_tets[j]] = 1;
                }
        std::fill(nmark.begin(), nmark.end(), 0);
        for (int64_t e = 0; e < E; ++e) {
            if (!mark[e]) continue;
            g.local_tets[p].push_back((int32_t)e);
            g.layer1[p].push_back(mark[e] == 2);
            for (int a = 0; a < 4; ++a) nmark[tet[4 * e + a]] = 1;
        }
        for (int64_t k = 0; k < N; ++k)
            if (nmark[k] || (g.node_owner[k] == p && g.node_off[k + 1] == g.node_off[k])) g.local_nodes[p].push_back((int32_t)k);
    }
}

// exchange lists of rank p with every peer q (sorted by global id on both sides, so the
// packed buffers line up without any index exchange)
void build_exchange(const PartGlobal &g, int p, PartLocal &L) {
    const int P = g.P;
    L.rank = p;
    L.nranks = P;
    L.tet_global = g.local_tets[p];
    L.node_global = g.local_nodes[p];
    const int64_t El = L.tet_global.size(), Nl = L.node_global.size();
    L.tet_flag.assign(El, 0);
    for (int64_t i = 0; i < El; ++i) {
        const int32_t e = L.tet_global[i];
        L.tet_flag[i] = (g.layer1[p][i] ? 1 : 0) | (g.tet_owner[e] == p ? 2 : 0);
    }
    L.node_owned.assign(Nl, 0);
    for (int64_t i = 0; i < Nl; ++i) L.node_owned[i] = g.node_owner[L.node_global[i]] == p;
    L.peers.clear();
    L.send_nodes.clear();
    L.recv_nodes.clear();
    L.send_tets.clear();
    L.recv_tets.clear();
    for (int q = 0; q < P; ++q) {
        if (q == p) continue;
        std::vector<int32_t> sn, rn, st, rt;
        // nodes owned by p that q holds (send), nodes owned by q that p holds (recv)
        {
            const auto &qn = g.local_nodes[q];
            for (size_t i = 0; i < qn.size(); ++i)
                if (g.node_owner[qn[i]] == p)
                    sn.push_back((int32_t)(std::lower_bound(L.node_global.begin(), L.node_global.end(), qn[i]) -
                                           L.node_global.begin()));
            for (int64_t i = 0; i < Nl; ++i)
                if (g.node_owner[L.node_global[i]] == q) rn.push_back((int32_t)i);
        }
        // tets owned by p that q holds as ghosts (send), tets owned by q that p holds as ghosts (recv)
        {
            const auto &qt = g.local_tets[q];
            for (size_t i = 0; i < qt.size(); ++i)
                if (!g.layer1[q][i] && g.tet_owner[qt[i]] == p)
                    st.push_back((int32_t)(std::lower_bound(L.tet_global.begin(), L.tet_global.end(), qt[i]) -
                                           L.tet_global.begin()));
            for (int64_t i = 0; i < El; ++i)
                if (!g.layer1[p][i] && g.tet_owner[L.tet_global[i]] == q) rt.push_back((int32_t)i);
        }
        if (sn.empty() && rn.empty() && st.empty() && rt.empty()) continue;
        L.peers.push_back(q);
        L.send_nodes.push_back(sn);
        L.recv_nodes.push_back(rn);
        L.send_tets.push_back(st);
        L.recv_tets.push_back(rt);
    }
}

}  // namespace cem
