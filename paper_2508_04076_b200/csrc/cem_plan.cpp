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

#include <omp.h>

#include "cem_internal.h"

namespace cem {

namespace {

// ---------------------------------------------------------------- bank-aware row placement
// The stage kernels gather fp64 rows from shared-memory planes.  For 8-byte loads a half-warp
// (16 lanes) is served per pass; two lanes reading different rows r != r' with r = r' (mod 16)
// hit the same bank pair and serialise.  Given the groups of items one half-warp instruction
// reads together, colour every item with k = row mod 16 so that a group's items get distinct
// colours where possible (greedy, most-constrained item first, then a swap pass that lowers
// sum_g sum_k cnt[g][k]^2).  Colour capacities are exact, so rows stay 0..n-1; inside a colour
// items keep ascending order (gather locality).  Returns row[item].
#ifndef CEM_BANK_SWAP
#define CEM_BANK_SWAP 0  // swap passes after the greedy colouring (1: -0.3 us/step, +45 ms host time)
#endif
// reusable per-thread buffers of bank_rows (the plan calls it once per block)
struct BankScratch {
    std::vector<int32_t> moff, mem, f, cnt, col, cap, order, goff, gitem, row;
    std::vector<std::vector<int32_t>> byc;
};

void bank_rows(int n, const std::vector<int32_t> &goff, const std::vector<int32_t> &gitem, std::vector<int32_t> &row,
               BankScratch &w) {
    row.assign(n, 0);
    if (n <= 16) {
        std::iota(row.begin(), row.end(), 0);
        return;
    }
    const int ng = (int)goff.size() - 1;
    std::vector<int32_t> &moff = w.moff, &mem = w.mem;
    moff.assign(n + 1, 0);
    for (int g = 0; g < ng; ++g)
        for (int32_t i = goff[g]; i < goff[g + 1]; ++i) moff[gitem[i] + 1]++;
    for (int i = 0; i < n; ++i) moff[i + 1] += moff[i];
    mem.resize(moff[n]);
    {
        std::vector<int32_t> &f = w.f;
        f.assign(moff.begin(), moff.end() - 1);
        for (int g = 0; g < ng; ++g)
            for (int32_t i = goff[g]; i < goff[g + 1]; ++i) mem[f[gitem[i]]++] = g;
    }
    std::vector<int32_t> &cnt = w.cnt, &col = w.col, &cap = w.cap, &order = w.order;
    cnt.assign((size_t)ng * 16, 0);
    col.assign(n, -1);
    cap.assign(16, 0);
    for (int k = 0; k < 16; ++k) cap[k] = n / 16 + (k < n % 16 ? 1 : 0);
    // items by degree, descending, ties in index order (a stable counting sort)
    order.resize(n);
    {
        int dmax = 0;
        for (int i = 0; i < n; ++i) dmax = std::max(dmax, moff[i + 1] - moff[i]);
        std::vector<int32_t> &f = w.f;
        f.assign(dmax + 2, 0);
        for (int i = 0; i < n; ++i) f[dmax - (moff[i + 1] - moff[i]) + 1]++;
        for (int k = 0; k <= dmax; ++k) f[k + 1] += f[k];
        for (int i = 0; i < n; ++i) order[f[dmax - (moff[i + 1] - moff[i])]++] = i;
    }
    for (int it : order) {
        int best = -1;
        long bc = 0;
        for (int k = 0; k < 16; ++k) {
            if (!cap[k]) continue;
            long c = 0;
            for (int32_t j = moff[it]; j < moff[it + 1]; ++j) c += cnt[(size_t)mem[j] * 16 + k];
            c = c * 1024 - cap[k];
            if (best < 0 || c < bc) best = k, bc = c;
        }
        col[it] = best;
        cap[best]--;
        for (int32_t j = moff[it]; j < moff[it + 1]; ++j) cnt[(size_t)mem[j] * 16 + best]++;
    }
    // swap pass: move a to its best colour k, b (colour k) to a's colour, if the sum of squares drops
    std::vector<std::vector<int32_t>> &byc = w.byc;
    byc.resize(16);
    for (auto &v : byc) v.clear();
    for (int i = 0; i < n; ++i) byc[col[i]].push_back(i);
    auto move_delta = [&](int it, int from, int to) {  // change of sum cnt^2 when `it` moves
        long dd = 0;
        for (int32_t j = moff[it]; j < moff[it + 1]; ++j) {
            const int32_t *c = &cnt[(size_t)mem[j] * 16];
            dd += 2L * (c[to] - c[from] + 1);
        }
        return dd;
    };
    auto apply = [&](int it, int from, int to) {
        for (int32_t j = moff[it]; j < moff[it + 1]; ++j) {
            cnt[(size_t)mem[j] * 16 + from]--;
            cnt[(size_t)mem[j] * 16 + to]++;
        }
        col[it] = to;
    };
    for (int pass = 0; pass < CEM_BANK_SWAP; ++pass) {
        bool any = false;
        for (int a = 0; a < n; ++a) {
            const int ka = col[a];
            int kb = -1;
            long da = 0;
            for (int k = 0; k < 16; ++k) {
                if (k == ka) continue;
                const long d = move_delta(a, ka, k);
                if (kb < 0 || d < da) kb = k, da = d;
            }
            if (da >= 0) continue;
            apply(a, ka, kb);
            int bb = -1;
            long db = 0;
            for (int b : byc[kb]) {
                if (b == a) continue;
                const long d = move_delta(b, kb, ka);
                if (bb < 0 || d < db) bb = b, db = d;
            }
            if (bb >= 0 && da + db < 0) {
                apply(bb, kb, ka);
                auto &A = byc[ka], &B = byc[kb];
                A.erase(std::find(A.begin(), A.end(), a));
                B.erase(std::find(B.begin(), B.end(), bb));
                A.push_back(bb);
                B.push_back(a);
                any = true;
            } else {
                apply(a, kb, ka);  // undo
            }
        }
        if (!any) break;
    }
    for (int k = 0; k < 16; ++k) {
        auto &v = byc[k];
        std::sort(v.begin(), v.end());
        for (size_t q = 0; q < v.size(); ++q) row[v[q]] = (int32_t)(16 * q + k);
    }
}

// groups of the items read together: lanes [h0, h0+16) x column l of tab (row stride `stride`)
template <class T>
void half_warp_groups(const T *tab, int64_t lo, int64_t hi, int stride, int width, std::vector<int32_t> &goff,
                      std::vector<int32_t> &gitem, int skip = -1) {
    goff.assign(1, 0);
    gitem.clear();
    for (int64_t h0 = lo; h0 < hi; h0 += 16)
        for (int l = 0; l < width; ++l) {
            const size_t st = gitem.size();
            for (int64_t i = h0; i < std::min<int64_t>(hi, h0 + 16); ++i) {
                const int v = (int)tab[(int64_t)stride * i + l];
                if (v == skip) continue;
                // insertion into the group's sorted, duplicate-free run (<= 16 items)
                size_t j = gitem.size();
                bool dup = false;
                while (j > st && gitem[j - 1] >= v) {
                    if (gitem[j - 1] == v) dup = true;
                    --j;
                }
                if (!dup) gitem.insert(gitem.begin() + j, v);
            }
            goff.push_back((int32_t)gitem.size());
        }
}

// reorder list[off..off+n) so that item i moves to row[i]
template <class T>
void permute_rows(T *list, int n, const std::vector<int32_t> &row) {
    thread_local std::vector<T> tmp;
    tmp.assign(list, list + n);
    for (int i = 0; i < n; ++i) list[row[i]] = tmp[i];
}

// Deduplicate vals[0..n) into the ascending list `uniq` and report every entry's position in it
// through put(i, pos): one sort of (value, index) keys instead of a sort plus n binary searches.
template <class Put>
void dedupe(const int32_t *vals, int n, std::vector<int32_t> &uniq, std::vector<uint64_t> &scratch, Put put) {
    scratch.resize(n);
    for (int i = 0; i < n; ++i) scratch[i] = (uint64_t)(uint32_t)vals[i] << 32 | (uint32_t)i;
    std::sort(scratch.begin(), scratch.end());
    uniq.clear();
    uniq.reserve(n);
    for (int i = 0; i < n; ++i) {
        const int32_t v = (int32_t)(scratch[i] >> 32);
        if (uniq.empty() || uniq.back() != v) uniq.push_back(v);
        put((int)(uint32_t)scratch[i], (int)uniq.size() - 1);
    }
}

}  // namespace

void build_plan(const HostMesh &h, int blk, Plan &p, const uint8_t *tflag_orig, bool with_deps) {
    const int64_t N = h.N, E = h.E, S = h.S;
    p.blk = blk;
    p.blk_ab = CEM_AB_EPT * blk;
    if (const char *ea = getenv("CEM_AB_EDGES")) p.blk_ab = std::max(blk, atoi(ea));  // (edges per AB block)
    const int blk_ab = p.blk_ab;
    PhaseClock clk;
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
#pragma omp parallel for schedule(static)
    for (int64_t e = 0; e < E; ++e) {
        for (int c = 0; c < 3; ++c) {
            double x = 0.0;
            for (int a = 0; a < 4; ++a) x += h.X[3 * (int64_t)h.tet[4 * e + a] + c];
            cen[3 * e + c] = 0.25 * x;
        }
        key[e] = (int64_t)std::floor((cen[3 * e + ax] - lo[ax]) / (kSlab * hb));
    }
    // tets by slab key, ascending id inside a slab (a stable counting sort, parallel)
    p.tet_new2old.resize(E);
    {
        int64_t kmax = 0;
        for (int64_t e = 0; e < E; ++e) kmax = std::max(kmax, key[e]);
        const int nk = (int)kmax + 1;
        const int nth = omp_get_max_threads();
        std::vector<int64_t> cnt((size_t)nth * nk + 1, 0);  // [thread][key] -> start
#pragma omp parallel num_threads(nth)
        {
            const int t = omp_get_thread_num();
            const int64_t e0 = E * t / nth, e1 = E * (t + 1) / nth;
            for (int64_t e = e0; e < e1; ++e) cnt[(size_t)t * nk + key[e]]++;
#pragma omp barrier
#pragma omp single
            {
                int64_t acc = 0;
                for (int k = 0; k < nk; ++k)
                    for (int tt = 0; tt < nth; ++tt) {
                        const int64_t c = cnt[(size_t)tt * nk + k];
                        cnt[(size_t)tt * nk + k] = acc;
                        acc += c;
                    }
            }
            for (int64_t e = e0; e < e1; ++e) p.tet_new2old[cnt[(size_t)t * nk + key[e]]++] = (int32_t)e;
        }
    }
    {
        const int64_t leaf = std::max(1, blk / 2);
        std::vector<int64_t> slab0;  // slab boundaries in the key-sorted order
        for (int64_t i = 0; i < E; ++i)
            if (i == 0 || key[p.tet_new2old[i]] != key[p.tet_new2old[i - 1]]) slab0.push_back(i);
        slab0.push_back(E);
        const int64_t nslab = (int64_t)slab0.size() - 1;
#pragma omp parallel for schedule(dynamic, 1)
        for (int64_t sl = 0; sl < nslab; ++sl) {  // slabs are independent
            std::vector<std::pair<int64_t, int64_t>> stack;
            const int64_t i0 = slab0[sl], i1 = slab0[sl + 1];
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
        }
    }
    clk.mark("plan: tet order");
    // nodes and edges by first appearance in the tet storage order: position of an entity =
    // min over its incidences of (new tet index, local index); entities sorted by it (a
    // compaction over the positions), entities referenced by no tet last in original order
    p.tet_old2new.assign(E, -1);
#pragma omp parallel for schedule(static)
    for (int64_t e = 0; e < E; ++e) p.tet_old2new[p.tet_new2old[e]] = (int32_t)e;
    std::vector<int32_t> edge_old2new(S, -1);
    auto number = [&](int64_t n, int per, auto first_pos, std::vector<int32_t> &old2new, std::vector<int32_t> &new2old) {
        std::vector<int32_t> at((size_t)per * E, -1);  // position -> entity
        std::vector<uint8_t> unused(n, 0);
#pragma omp parallel for schedule(static)
        for (int64_t k = 0; k < n; ++k) {
            const int64_t fp = first_pos(k);
            if (fp >= 0) at[fp] = (int32_t)k;
            else unused[k] = 1;
        }
        const int nth = omp_get_max_threads();
        const int64_t P = (int64_t)per * E;
        std::vector<int64_t> base(nth + 1, 0);
        new2old.resize(n);
        old2new.assign(n, -1);
#pragma omp parallel num_threads(nth)
        {
            const int t = omp_get_thread_num();
            const int64_t i0 = P * t / nth, i1 = P * (t + 1) / nth;
            int64_t c = 0;
            for (int64_t i = i0; i < i1; ++i) c += at[i] >= 0;
            base[t + 1] = c;
#pragma omp barrier
#pragma omp single
            for (int tt = 0; tt < nth; ++tt) base[tt + 1] += base[tt];
            int64_t j = base[t];
            for (int64_t i = i0; i < i1; ++i)
                if (at[i] >= 0) {
                    new2old[j] = at[i];
                    old2new[at[i]] = (int32_t)j;
                    ++j;
                }
        }
        int64_t j = base[nth];
        for (int64_t k = 0; k < n; ++k)
            if (unused[k]) {
                new2old[j] = (int32_t)k;
                old2new[k] = (int32_t)j++;
            }
    };
    number(N, 4, [&](int64_t k) -> int64_t {
        int64_t best = -1;
        for (int32_t i = h.node_off[k]; i < h.node_off[k + 1]; ++i) {
            const int32_t ent = h.node_ent[i];
            const int64_t pos = 4 * (int64_t)p.tet_old2new[ent >> 2] + (ent & 3);
            if (best < 0 || pos < best) best = pos;
        }
        return best;
    }, p.node_old2new, p.node_new2old);
    number(S, 6, [&](int64_t s) -> int64_t {
        int64_t best = -1;
        for (int32_t i = h.edge_off[s]; i < h.edge_off[s + 1]; ++i) {
            const int32_t eo = h.edge_inc[i];
            int l = 0;
            while (h.elem_edge[6 * (int64_t)eo + l] != (int32_t)s) ++l;
            const int64_t pos = 6 * (int64_t)p.tet_old2new[eo] + l;
            if (best < 0 || pos < best) best = pos;
        }
        return best;
    }, edge_old2new, p.edge_new2old);
    clk.mark("plan: node/edge order");
    // ---------------------------------------------------------------- storage-order tables
    p.conn.resize(4 * E);
    p.geoV.resize(E);
    p.geoC.resize(E);
    // geometry records written straight into the device layout (CEM_GEO_AOS)
#if CEM_GEO_AOS
    p.geoT.resize((size_t)E * 12);  // per tet 12 doubles (96 B): V, V/6, gradN1..3 (x, y, z), (pad)
#else
    p.geoT.resize((size_t)((E + 31) / 32) * 11 * 32);  // [E/32][11][32] warp tiles (tail lanes unused)
#endif
    p.eedge.resize(6 * E);
    p.state.resize(E);
    p.tflag.resize(E);
    p.gc.resize(E);
#pragma omp parallel for schedule(static)
    for (int64_t en = 0; en < E; ++en) {
        const int64_t eo = p.tet_new2old[en];
        for (int a = 0; a < 4; ++a) p.conn[4 * en + a] = p.node_old2new[h.tet[4 * eo + a]];
        p.geoV[en] = h.V[eo];
        p.geoC[en] = h.V[eo] / 6.0;
#if CEM_GEO_AOS
        double *g = p.geoT.data() + 12 * en;
        const int gs = 1;
#else
        double *g = p.geoT.data() + (en >> 5) * 352 + (en & 31);
        const int gs = 32;
#endif
        g[0] = p.geoV[en];
        g[gs] = p.geoC[en];
        for (int a = 1; a < 4; ++a)
            for (int c = 0; c < 3; ++c) g[gs * (2 + 3 * (a - 1) + c)] = h.grad[12 * eo + 3 * a + c];
        for (int l = 0; l < 6; ++l) p.eedge[(int64_t)l * E + en] = edge_old2new[h.elem_edge[6 * eo + l]];
        p.state[en] = h.state[eo];
        p.tflag[en] = tflag_orig ? tflag_orig[eo] : 3;
        p.gc[en] = h.gc[eo];
    }
    p.edge_off.assign(S + 1, 0);
    for (int64_t sn = 0; sn < S; ++sn) {
        const int32_t so = p.edge_new2old[sn];
        p.edge_off[sn + 1] = p.edge_off[sn] + (h.edge_off[so + 1] - h.edge_off[so]);
    }
    p.edge_inc.resize(h.edge_inc.size());
#pragma omp parallel for schedule(static)
    for (int64_t sn = 0; sn < S; ++sn) {
        const int32_t so = p.edge_new2old[sn];
        int32_t j = p.edge_off[sn];
        for (int32_t i = h.edge_off[so]; i < h.edge_off[so + 1]; ++i) p.edge_inc[j++] = p.tet_old2new[h.edge_inc[i]];
    }
    p.node_off.assign(N + 1, 0);
    for (int64_t kn = 0; kn < N; ++kn) {
        const int32_t ko = p.node_new2old[kn];
        p.node_off[kn + 1] = p.node_off[kn] + (h.node_off[ko + 1] - h.node_off[ko]);
    }
    p.node_ent.resize(h.node_ent.size());
#pragma omp parallel for schedule(static)
    for (int64_t kn = 0; kn < N; ++kn) {
        const int32_t ko = p.node_new2old[kn];
        int32_t j = p.node_off[kn];
        for (int32_t i = h.node_off[ko]; i < h.node_off[ko + 1]; ++i) {
            const int32_t ent = h.node_ent[i];
            p.node_ent[j++] = (p.tet_old2new[ent >> 2] << 2) | (ent & 3);
        }
    }
    clk.mark("plan: storage tables");
    // ---------------------------------------------------------------- gather lists
    {
        const int nbt = (int)((E + blk - 1) / blk), nbs = (int)((S + blk_ab - 1) / blk_ab);
        // per-block lists built in parallel, then concatenated
        auto concat = [](std::vector<std::vector<int32_t>> &parts, std::vector<int32_t> &off, std::vector<int32_t> &out,
                         int &mx) {
            off.assign(parts.size() + 1, 0);
            mx = 0;
            for (size_t b = 0; b < parts.size(); ++b) {
                off[b + 1] = off[b] + (int32_t)parts[b].size();
                mx = std::max(mx, (int)parts[b].size());
            }
            out.resize(off.back());
#pragma omp parallel for schedule(static)
            for (int64_t b = 0; b < (int64_t)parts.size(); ++b) std::copy(parts[b].begin(), parts[b].end(), out.begin() + off[b]);
        };
        p.lconn.resize(4 * E);  // (written in full below)
        p.ledge.resize(8 * E);  // (6 of 8 written per tet; the rest is never read)
        {
            std::vector<std::vector<int32_t>> nlv(nbt), elv(nbt);
#pragma omp parallel
            {
                std::vector<uint64_t> scratch;
                std::vector<int32_t> vals;
#pragma omp for schedule(dynamic, 16)
                for (int b = 0; b < nbt; ++b) {
                    const int64_t e0 = (int64_t)b * blk, e1 = std::min<int64_t>(E, e0 + blk);
                    const int n = (int)(e1 - e0);
                    dedupe(p.conn.data() + 4 * e0, 4 * n, nlv[b], scratch,
                           [&](int i, int pos) { p.lconn[4 * e0 + i] = (uint16_t)pos; });
                    vals.resize(6 * n);
                    for (int i = 0; i < n; ++i)
                        for (int l = 0; l < 6; ++l) vals[6 * i + l] = p.eedge[(int64_t)l * E + e0 + i];
                    dedupe(vals.data(), 6 * n, elv[b], scratch,
                           [&](int i, int pos) { p.ledge[8 * (e0 + i / 6) + i % 6] = (uint16_t)pos; });
                }
            }
            concat(nlv, p.nl_off, p.nl, p.max_nl);
            concat(elv, p.el_off, p.el, p.max_el);
        }
        p.inc_local.resize(p.edge_inc.size());  // (written in full below)
        {
            std::vector<std::vector<int32_t>> tlv(nbs);
#pragma omp parallel
            {
                std::vector<uint64_t> scratch;
#pragma omp for schedule(dynamic, 16)
                for (int b = 0; b < nbs; ++b) {
                    const int64_t s0 = (int64_t)b * blk_ab, s1 = std::min<int64_t>(S, s0 + blk_ab);
                    const int32_t j0 = p.edge_off[s0];
                    dedupe(p.edge_inc.data() + j0, p.edge_off[s1] - j0, tlv[b], scratch,
                           [&](int i, int pos) { p.inc_local[j0 + i] = (uint16_t)pos; });
                }
            }
            concat(tlv, p.tl_off, p.tl, p.max_tl);
        }
        clk.mark("plan: gather lists");
        // bank-aware order of each edge block's tet list: lanes = edges, column t = t-th incidence
        {
            std::vector<uint16_t> incw((size_t)S * 8, 0xFFFF);  // first 8 incidences per edge (ELL view)
#pragma omp parallel for schedule(static)
            for (int64_t s = 0; s < S; ++s)
                for (int32_t j = p.edge_off[s]; j < std::min(p.edge_off[s + 1], p.edge_off[s] + 8); ++j)
                    incw[8 * s + (j - p.edge_off[s])] = p.inc_local[j];
            int wmax = 1;
            for (int64_t s = 0; s < S; ++s) wmax = std::max(wmax, p.edge_off[s + 1] - p.edge_off[s]);
            wmax = std::min(wmax, 8);
            p.trow.assign(p.tl.size(), 0);
#pragma omp parallel
            {
                BankScratch w;
                std::vector<int32_t> &goff = w.goff, &gitem = w.gitem, &row = w.row;
#pragma omp for schedule(dynamic, 16)
                for (int b = 0; b < nbs; ++b) {
                    const int64_t s0 = (int64_t)b * blk_ab, s1 = std::min<int64_t>(S, s0 + blk_ab);
                    const int nt = p.tl_off[b + 1] - p.tl_off[b];
                    half_warp_groups(incw.data(), s0, s1, 8, wmax, goff, gitem, 0xFFFF);
                    bank_rows(nt, goff, gitem, row, w);
                    // the list keeps ascending tet order (thread i gathers entry i: coalesced); entry i
                    // writes its tau into shared-memory row trow[i]
                    for (int i = 0; i < nt; ++i) p.trow[p.tl_off[b] + i] = (uint16_t)row[i];
                    for (int32_t j = p.edge_off[s0]; j < p.edge_off[s1]; ++j) p.inc_local[j] = (uint16_t)row[p.inc_local[j]];
                }
            }
        }
        clk.mark("plan: bank order (tets)");
        // nodes of each edge block's tet list (the fused AB stage recomputes tau from them)
        p.tconn.resize(4 * p.tl.size());  // (written in full below)
        {
            std::vector<std::vector<int32_t>> nbv(nbs);
#pragma omp parallel
            {
                std::vector<uint64_t> scratch;
                std::vector<int32_t> vals;
#pragma omp for schedule(dynamic, 16)
                for (int b = 0; b < nbs; ++b) {
                    const int32_t t0 = p.tl_off[b], nt = p.tl_off[b + 1] - t0;
                    vals.resize(4 * (size_t)nt);
                    for (int32_t i = 0; i < nt; ++i)
                        for (int a = 0; a < 4; ++a) vals[4 * i + a] = p.conn[4 * (int64_t)p.tl[t0 + i] + a];
                    dedupe(vals.data(), 4 * nt, nbv[b], scratch,
                           [&](int i, int pos) { p.tconn[4 * (int64_t)t0 + i] = (uint16_t)pos; });
                }
            }
            concat(nbv, p.nlb_off, p.nlb, p.max_nlb);
        }
        clk.mark("plan: AB node lists");
        // bank-aware order of the staged node lists: AB (lanes = tet-list rows, column a) and
        // C's early-out (lanes = tets, column a); C's edge lists (lanes = tets, column l)
        p.nrow.assign(p.nlb.size(), 0);
#pragma omp parallel
        {
            BankScratch w;
            std::vector<int32_t> &goff = w.goff, &gitem = w.gitem, &row = w.row;
#pragma omp for schedule(dynamic, 16) nowait
            for (int b = 0; b < nbs; ++b) {
                const int32_t t0 = p.tl_off[b];
                const int nt = p.tl_off[b + 1] - t0, nn = p.nlb_off[b + 1] - p.nlb_off[b];
                half_warp_groups(p.tconn.data() + 4 * (int64_t)t0, 0, nt, 4, 4, goff, gitem);
                bank_rows(nn, goff, gitem, row, w);
                for (int i = 0; i < nn; ++i) p.nrow[p.nlb_off[b] + i] = (uint16_t)row[i];  // staging row of entry i
                for (int64_t i = 4 * (int64_t)t0; i < 4 * (int64_t)(t0 + nt); ++i) p.tconn[i] = (uint16_t)row[p.tconn[i]];
            }
#pragma omp for schedule(dynamic, 16)
            for (int b = 0; b < nbt; ++b) {
                const int64_t e0 = (int64_t)b * blk, e1 = std::min<int64_t>(E, e0 + blk);
                const int ne = p.el_off[b + 1] - p.el_off[b], nn = p.nl_off[b + 1] - p.nl_off[b];
                half_warp_groups(p.ledge.data(), e0, e1, 8, 6, goff, gitem);
                bank_rows(ne, goff, gitem, row, w);
                permute_rows(p.el.data() + p.el_off[b], ne, row);
                for (int64_t e = e0; e < e1; ++e)
                    for (int l = 0; l < 6; ++l) p.ledge[8 * e + l] = (uint16_t)row[p.ledge[8 * e + l]];
                half_warp_groups(p.lconn.data(), e0, e1, 4, 4, goff, gitem);
                bank_rows(nn, goff, gitem, row, w);
                permute_rows(p.nl.data() + p.nl_off[b], nn, row);
                for (int64_t i = 4 * e0; i < 4 * e1; ++i) p.lconn[i] = (uint16_t)row[p.lconn[i]];
            }
        }
        clk.mark("plan: bank order (nodes, edges)");
    }
    // ---------------------------------------------------------------- exact partials (R27)
    // partial q = entry q of a stage-C block's node list (final, bank-permuted order): its
    // incidences among the block's tets as a blk + t (t local tet, a corner: stage C's force row)
    // in pinc[pinc_off[q] ..);
    // block b's entries fill pinc[4 e0, 4 e1) of its tet range.  Records are node-major: partial q
    // goes to record pdst[q], node k's records are [poff[k], poff[k+1]) (ascending block).
    {
        const char *ev = getenv("CEM_PARTIALS");
        p.partials = !(ev && atoi(ev) == 0);
        const int nbt = (int)((E + blk - 1) / blk);
        const int64_t NP = (int64_t)p.nl.size();
        p.pinc_off.resize(NP + 1);
        p.pinc.resize(4 * E);
#pragma omp parallel
        {
            std::vector<int32_t> cnt, fill;
#pragma omp for schedule(dynamic, 16)
            for (int b = 0; b < nbt; ++b) {
                const int64_t e0 = (int64_t)b * blk, e1 = std::min<int64_t>(E, e0 + blk);
                const int32_t n0 = p.nl_off[b], nn = p.nl_off[b + 1] - n0;
                cnt.assign(nn + 1, 0);
                for (int64_t i = 4 * e0; i < 4 * e1; ++i) cnt[p.lconn[i] + 1]++;
                for (int i = 0; i < nn; ++i) cnt[i + 1] += cnt[i];
                for (int i = 0; i < nn; ++i) p.pinc_off[n0 + i] = (int32_t)(4 * e0 + cnt[i]);
                fill.assign(cnt.begin(), cnt.end() - 1);
                for (int64_t e = e0; e < e1; ++e)
                    for (int a = 0; a < 4; ++a)  // stage C's shared-memory force row of (t, a): a blk + t
                        p.pinc[4 * e0 + fill[p.lconn[4 * e + a]]++] = (uint16_t)(a * blk + (e - e0));
            }
        }
        p.pinc_off[NP] = (int32_t)(4 * E);
        // per block, its entries by descending incidence count (a warp's 32 lanes then loop
        // over nearly equal counts)
        p.pord.resize(NP);
#pragma omp parallel for schedule(dynamic, 16)
        for (int b = 0; b < nbt; ++b) {
            const int32_t n0 = p.nl_off[b], nn = p.nl_off[b + 1] - n0;
            int32_t *o = p.pord.data() + n0;
            for (int i = 0; i < nn; ++i) o[i] = i;
            std::stable_sort(o, o + nn, [&](int32_t x, int32_t y) {
                return p.pinc_off[n0 + x + 1] - p.pinc_off[n0 + x] > p.pinc_off[n0 + y + 1] - p.pinc_off[n0 + y];
            });
            // bank-aware order inside each entry's incidence list: the 32 lanes of a warp (32
            // consecutive entries of o) read their u-th incidences together; force row a blk + t
            // sits at bank position t mod 16 of the f_z plane (t mod 8 of the (x, y) plane), so
            // step u greedily gives each lane the remaining incidence of the least-used position
            for (int w0 = 0; w0 < nn; w0 += 32) {
                const int w1 = std::min(nn, w0 + 32);
                int mxc = 0;
                for (int k = w0; k < w1; ++k) mxc = std::max(mxc, p.pinc_off[n0 + o[k] + 1] - p.pinc_off[n0 + o[k]]);
                for (int u = 0; u < mxc; ++u) {
                    int used[16] = {0};
                    for (int k = w0; k < w1; ++k) {
                        const int32_t j0 = p.pinc_off[n0 + o[k]], j1 = p.pinc_off[n0 + o[k] + 1];
                        if (j0 + u >= j1) continue;
                        int best = j0 + u;
                        for (int j = j0 + u + 1; j < j1; ++j)
                            if (used[(p.pinc[j] % blk) & 15] < used[(p.pinc[best] % blk) & 15]) best = j;
                        std::swap(p.pinc[j0 + u], p.pinc[best]);
                        ++used[(p.pinc[j0 + u] % blk) & 15];
                    }
                }
            }
        }
        // node-major records: node k's partials (ascending q, i.e. ascending block) are consecutive
        p.poff.assign(N + 1, 0);
        for (int64_t q = 0; q < NP; ++q) p.poff[p.nl[q] + 1]++;
        for (int64_t k = 0; k < N; ++k) p.poff[k + 1] += p.poff[k];
        p.pdst.resize(NP);
        std::vector<int32_t> fk(p.poff.begin(), p.poff.end() - 1);
        for (int64_t q = 0; q < NP; ++q) p.pdst[q] = fk[p.nl[q]]++;
        clk.mark("plan: partials");
        if (clk.on)
            fprintf(stderr, "[cem timing] blocks: max_el %d max_nl %d max_tl %d max_nlb %d partials %zu\n",
                    p.max_el, p.max_nl, p.max_tl, p.max_nlb, p.nl.size());
    }
    // ---------------------------------------------------------------- instruction-lean layouts
    {
        int mx = 1;
        for (int64_t s = 0; s < S; ++s) mx = std::max(mx, p.edge_off[s + 1] - p.edge_off[s]);
        p.we = (mx + 7) / 8 * 8;
        p.we_max = mx;
        p.incE.resize((size_t)S * p.we);
#pragma omp parallel for schedule(static)
        for (int64_t s = 0; s < S; ++s) {
            const int32_t n = p.edge_off[s + 1] - p.edge_off[s];
            for (int32_t j = 0; j < n; ++j) p.incE[(size_t)s * p.we + j] = p.inc_local[p.edge_off[s] + j];
            for (int32_t j = n; j < p.we; ++j) p.incE[(size_t)s * p.we + j] = 0xFFFF;
        }
        mx = 1;
        for (int64_t k = 0; k < N; ++k) mx = std::max(mx, p.node_off[k + 1] - p.node_off[k]);
        p.wn = (mx + 7) / 8 * 8;
        p.zslot = (int32_t)(((E + 31) / 32) * 128);  // first slot past the last tile: kept zero
        p.nodeE.resize((size_t)N * p.wn);
#pragma omp parallel for schedule(static)
        for (int64_t k = 0; k < N; ++k) {
            for (int32_t j = p.node_off[k + 1] - p.node_off[k]; j < p.wn; ++j) p.nodeE[(size_t)k * p.wn + j] = p.zslot;
            for (int32_t j = p.node_off[k]; j < p.node_off[k + 1]; ++j) {
                const int64_t e = p.node_ent[j] >> 2, a = p.node_ent[j] & 3;
#if CEM_FES == 3
                p.nodeE[(size_t)k * p.wn + (j - p.node_off[k])] = (int32_t)(4 * e + a);  // packed per tet
#else
                p.nodeE[(size_t)k * p.wn + (j - p.node_off[k])] = (int32_t)((((e >> 5) * 4 + a) << 5) + (e & 31));
#endif
            }
        }
    }
    clk.mark("plan: ELL tables");
    // ---------------------------------------------------------------- blocks and dependencies
    const int64_t cnt[ST_COUNT] = {S, E, N};
    const int per[ST_COUNT] = {blk_ab, blk, blk};
    p.maxblk = 0;
    for (int g = 0; g < ST_COUNT; ++g) {
        p.nblk[g] = (int)((cnt[g] + per[g] - 1) / per[g]);
        p.maxblk = std::max(p.maxblk, p.nblk[g]);
    }
    if (!with_deps) {  // the producer lists serve only the persistent wavefront kernel
        p.dep_off.clear();
        p.dep.clear();
        p.ncons.clear();
        return;
    }
    // explicit producer-block lists per (stage, block)
    std::vector<std::vector<int32_t>> deps((size_t)ST_COUNT * p.maxblk);
    auto finish = [](std::vector<int32_t> &v) {
        std::sort(v.begin(), v.end());
        v.erase(std::unique(v.begin(), v.end()), v.end());
    };
#pragma omp parallel for schedule(dynamic, 64)
    for (int b = 0; b < p.nblk[ST_AB]; ++b) {  // AB: D-blocks (previous step) of its tet list's nodes
        auto &v = deps[(size_t)ST_AB * p.maxblk + b];
        for (int32_t i = p.nlb_off[b]; i < p.nlb_off[b + 1]; ++i) v.push_back(p.nlb[i] / blk);
        finish(v);
    }
#pragma omp parallel for schedule(dynamic, 64)
    for (int b = 0; b < p.nblk[ST_C]; ++b) {  // C: AB-blocks of its edge list
        auto &v = deps[(size_t)ST_C * p.maxblk + b];
        for (int32_t i = p.el_off[b]; i < p.el_off[b + 1]; ++i) v.push_back(p.el[i] / blk_ab);
        finish(v);
    }
#pragma omp parallel for schedule(dynamic, 64)
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
    }    clk.mark("plan: dependencies");
}

// K chunks of stage-C blocks; chunk c is preceded by the AB blocks its edges need that earlier
// chunks did not already launch (AB blocks of the edges of C blocks [0, c1) = prefix max)
std::vector<StageChunk> build_stage_chunks(const Plan &p, int K) {
    std::vector<StageChunk> out;
    const int nC = p.nblk[ST_C], nAB = p.nblk[ST_AB];
    K = std::max(1, std::min(K, nC));
    int a = 0, m = -1, b = 0;
    for (int c = 0; c < K; ++c) {
        const int c1 = (int)((int64_t)nC * (c + 1) / K);
        for (; b < c1; ++b)
            for (int32_t i = p.el_off[b]; i < p.el_off[b + 1]; ++i) m = std::max(m, p.el[i] / p.blk_ab);
        const int a1 = c + 1 == K ? nAB : std::max(a, m + 1);
        out.push_back({a, a1, (int)((int64_t)nC * c / K), c1});
        a = a1;
    }
    return out;
}

void build_wave(const Plan &p, int64_t N, int chunks, int lookahead, WavePlan &w) {
    const int nAB = p.nblk[ST_AB], nC = p.nblk[ST_C], nD = (int)((N + kDW - 1) / kDW);
    w.nblk[ST_AB] = nAB;
    w.nblk[ST_C] = nC;
    w.nblk[ST_D] = nD;
    w.maxblk = std::max(nAB, std::max(nC, nD));
    std::vector<std::vector<int32_t>> deps((size_t)ST_COUNT * w.maxblk);
    auto finish = [](std::vector<int32_t> &v) {
        std::sort(v.begin(), v.end());
        v.erase(std::unique(v.begin(), v.end()), v.end());
    };
#pragma omp parallel for schedule(dynamic, 64)
    for (int b = 0; b < nAB; ++b) {  // AB: the D blocks (previous step) of its tet list's nodes
        auto &v = deps[(size_t)ST_AB * w.maxblk + b];
        for (int32_t i = p.nlb_off[b]; i < p.nlb_off[b + 1]; ++i) v.push_back(p.nlb[i] / kDW);
        finish(v);
    }
#pragma omp parallel for schedule(dynamic, 64)
    for (int b = 0; b < nC; ++b) {  // C: the AB blocks of its edge list
        auto &v = deps[(size_t)ST_C * w.maxblk + b];
        for (int32_t i = p.el_off[b]; i < p.el_off[b + 1]; ++i) v.push_back(p.el[i] / p.blk_ab);
        finish(v);
    }
#pragma omp parallel for schedule(dynamic, 64)
    for (int b = 0; b < nD; ++b) {  // D: the C blocks of the tets of its nodes
        auto &v = deps[(size_t)ST_D * w.maxblk + b];
        for (int64_t k = (int64_t)b * kDW; k < std::min<int64_t>(N, (int64_t)(b + 1) * kDW); ++k)
            for (int32_t j = p.node_off[k]; j < p.node_off[k + 1]; ++j) v.push_back((p.node_ent[j] >> 2) / p.blk);
        finish(v);
    }
    w.ncons.assign((size_t)2 * w.maxblk, 0);
    for (int g = ST_C; g <= ST_D; ++g)
        for (int b = 0; b < w.nblk[g]; ++b)
            for (int32_t pb : deps[(size_t)g * w.maxblk + b]) w.ncons[(size_t)(g - 1) * w.maxblk + pb]++;
    w.dep_off.assign((size_t)ST_COUNT * w.maxblk + 1, 0);
    w.dep.clear();
    for (size_t q = 0; q < deps.size(); ++q) {
        w.dep.insert(w.dep.end(), deps[q].begin(), deps[q].end());
        w.dep_off[q + 1] = (int32_t)w.dep.size();
    }
    // launch sequence: K chunks of C blocks; before C chunk c the AB blocks that C chunks up to
    // c + lookahead read; after it the D blocks whose C producers lie in chunks <= c - lookahead
    const int K = std::max(1, std::min(chunks, nC));
    auto maxdep = [&](int g, int b) {
        const size_t q = (size_t)g * w.maxblk + b;
        return w.dep_off[q + 1] > w.dep_off[q] ? w.dep[w.dep_off[q + 1] - 1] : -1;
    };
    std::vector<int> cend(K);  // C chunk c = [cend[c-1], cend[c])
    for (int c = 0; c < K; ++c) cend[c] = (int)((int64_t)nC * (c + 1) / K);
    std::vector<int> abneed(K);  // AB blocks [0, abneed[c]) cover C chunks <= c (prefix max)
    {
        int m = -1, b = 0;
        for (int c = 0; c < K; ++c) {
            for (; b < cend[c]; ++b) m = std::max(m, maxdep(ST_C, b));
            abneed[c] = m + 1;
        }
    }
    std::vector<int> dpref(nD);  // prefix max of the largest C producer of D blocks [0, b]
    {
        int m = -1;
        for (int b = 0; b < nD; ++b) dpref[b] = m = std::max(m, maxdep(ST_D, b));
    }
    w.seq.clear();
    int a = 0, dd = 0;
    auto emit = [&](int g, int b0, int b1) {
        if (b1 > b0) w.seq.push_back({g, b0, b1});
    };
    for (int c = 0; c < K; ++c) {
        const int an = std::max(abneed[std::min(K - 1, c + lookahead)], c + 1 == K ? nAB : 0);
        if (an > a) {
            emit(ST_AB, a, an);
            a = an;
        }
        emit(ST_C, c ? cend[c - 1] : 0, cend[c]);
        const int cc = c - lookahead;  // D blocks whose producers are all in C chunks <= cc
        if (cc >= 0) {
            int d1 = dd;
            while (d1 < nD && dpref[d1] < cend[cc]) ++d1;
            emit(ST_D, dd, d1);
            dd = d1;
        }
    }
    if (a < nAB) emit(ST_AB, a, nAB);  // (edges of no tet: none in a valid mesh)
    for (int cc = std::max(0, K - lookahead); cc < K; ++cc) {  // the remaining D blocks
        int d1 = dd;
        while (d1 < nD && dpref[d1] < cend[cc]) ++d1;
        emit(ST_D, dd, d1);
        dd = d1;
    }
    emit(ST_D, dd, nD);
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
