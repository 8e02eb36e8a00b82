// cem_hex.cu -- sm_100a kernels of the ES-H-FEM step on trilinear hexahedra (
// PAPER.md:L311-L338 eq:hex_strain_discretization, L368-L390 eq:hex_fint_discretization).
// Same bitwise contract as the tet path (--fmad=false, sequential sums in the order of
// DESIGN.md §5 for hexes).  Crack patterns III-VI (R28): a split hex may leave a remainder of three
// tets (E + 3e + i) over its own nodes; their data sit with the parent hex.
//   A  tau_e = V_e eps_e, eps from the mean gradients (R23), a = 0..7      -> 32-B + 16-B record planes;
//      remainder tets tau = V_t eps_t over their 4 nodes                    -> [E][3][6]
//   B  sigma_s = D (sum tau) / (sum V) over the active elements of edge s (hex e, then its
//      remainder tets; R29), edges [0, S_h) hex edges, [S_h, S) diagonals
//   C  S_e = sum_{l=0..11} sigma_{s(e,l)}; f_{e,a} = (V_e/12) B_a^T S_e (R26) -> slot 8e + a (192 B per hex);
//      remainder tet i: (V_t/6) B^T sum of its 6 edges -> slot 8E + 3(8e + a) + i of its nodes a
//   crit (crack steps, cem_kernels.cu k_hexcrit): patterns III-VI / the tet criterion, split
//   D  the tet path's node update (force-slot gather, Newmark, BC, mass of split nodes, predictor)
#include <cstdint>

#include "cem_internal.h"

namespace cem {

namespace {

__device__ __forceinline__ void pdl_trigger_h() { asm volatile("griddepcontrol.launch_dependents;" ::: "memory"); }
__device__ __forceinline__ void pdl_wait_h() { asm volatile("griddepcontrol.wait;" ::: "memory"); }
// 32-B / 16-B L2 loads and stores (one sector each: u of a node, the two planes of a tau record)
__device__ __forceinline__ double4 ldcg256h(const double4 *p) {
    double4 r;
    asm volatile("ld.global.cg.v4.f64 {%0,%1,%2,%3}, [%4];" : "=d"(r.x), "=d"(r.y), "=d"(r.z), "=d"(r.w) : "l"(p));
    return r;
}
__device__ __forceinline__ double2 ldcg128h(const double2 *p) {
    double2 r;
    asm volatile("ld.global.cg.v2.f64 {%0,%1}, [%2];" : "=d"(r.x), "=d"(r.y) : "l"(p));
    return r;
}
__device__ __forceinline__ void st256h(double4 *p, double x, double y, double z, double w) {
    asm volatile("st.global.v4.f64 [%0], {%1,%2,%3,%4};" ::"l"(p), "d"(x), "d"(y), "d"(z), "d"(w) : "memory");
}

// local node pair (a, b) -> 0..27 and the hex edge of a pair (-1: a face or body diagonal)
__constant__ int8_t c_hpair[8][8] = {{-1, 0, 1, 2, 3, 4, 5, 6},     {0, -1, 7, 8, 9, 10, 11, 12},
                                     {1, 7, -1, 13, 14, 15, 16, 17}, {2, 8, 13, -1, 18, 19, 20, 21},
                                     {3, 9, 14, 18, -1, 22, 23, 24}, {4, 10, 15, 19, 22, -1, 25, 26},
                                     {5, 11, 16, 20, 23, 25, -1, 27}, {6, 12, 17, 21, 24, 26, 27, -1}};
__constant__ int8_t c_hedge_of_pair[28] = {0,  -1, 3,  8, -1, -1, -1, 1, -1, -1, 9,  -1, -1, 2,
                                           -1, -1, 10, -1, -1, -1, -1, 11, 4, -1, 7, 5, -1, 6};
#ifndef CEM_HEXB_BATCH
#define CEM_HEXB_BATCH 2  // stage B: incidences gathered per pass (their loads in flight together; measured 1 / 2 / 4: 403 / 385 / 427 us per step on 100^3 hexes)
#endif
__constant__ int8_t c_tp[6] = {0, 0, 0, 1, 1, 2};
__constant__ int8_t c_tq[6] = {1, 2, 3, 2, 3, 3};

__device__ __forceinline__ bool tet_has_pair(const uint8_t *t, int pj) {
#pragma unroll
    for (int l = 0; l < 6; ++l)
        if (c_hpair[t[c_tp[l]]][t[c_tq[l]]] == pj) return true;
    return false;
}

__global__ void __launch_bounds__(256) k_hexA(Dev d, int64_t s) {
    pdl_trigger_h();
    const int64_t E = d.E;
    const int64_t e = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (e >= E) return;
    int32_t n[8];
#pragma unroll
    for (int a = 0; a < 8; ++a) n[a] = __ldg(d.hconn + a * E + e);
    const double V = __ldg(d.hgeo + e);
    double g[8][3];
#pragma unroll
    for (int a = 0; a < 8; ++a)
#pragma unroll
        for (int c = 0; c < 3; ++c) g[a][c] = __ldg(d.hgeo + (1 + 3 * a + c) * E + e);
    pdl_wait_h();  // u_{s+1} comes from the previous step's stage D
    const uint8_t act = __ldcg(d.state + e);
    const double4 *u = d.ubuf[(s + 1) & 1];
    double ex = 0.0, ey = 0.0, ez = 0.0, gxy = 0.0, gyz = 0.0, gxz = 0.0;
    if (act) {
#pragma unroll
        for (int a = 0; a < 8; ++a) {
            const double4 ua = ldcg256h(u + n[a]);
            const double ux = ua.x, uy = ua.y, uz = ua.z;
            ex = ex + g[a][0] * ux;
            ey = ey + g[a][1] * uy;
            ez = ez + g[a][2] * uz;
            gxy = gxy + (g[a][1] * ux + g[a][0] * uy);
            gyz = gyz + (g[a][2] * uy + g[a][1] * uz);
            gxz = gxz + (g[a][2] * ux + g[a][0] * uz);
        }
    }
    // tau record of hex e: (11, 22, 33, 12) as one 32-B record in plane [E], (23, 13) as one 16-B
    // record in the plane after it (stage B gathers a record with two loads instead of six)
    st256h(reinterpret_cast<double4 *>(d.htau) + e, act ? V * ex : 0.0, act ? V * ey : 0.0, act ? V * ez : 0.0,
           act ? V * gxy : 0.0);
    reinterpret_cast<double2 *>(d.htau + 4 * E)[e] = make_double2(act ? V * gyz : 0.0, act ? V * gxz : 0.0);
    if (__ldcg(d.hrem + e) < 0) return;
    const uint8_t ta = __ldcg(d.htact + e);
    for (int i = 0; i < 3; ++i) {
        double *tt = d.httau + 18 * e + 6 * i;
        if (!(ta >> i & 1)) continue;
        const uint8_t *tl = d.htloc + 12 * e + 4 * i;
        const double *tg = d.htgeo + 39 * e + 13 * i;
        double x = 0.0, y = 0.0, z = 0.0, xy = 0.0, yz = 0.0, xz = 0.0;
        for (int a = 0; a < 4; ++a) {
            const double4 ua = ldcg256h(u + n[tl[a]]);
            const double ux = ua.x, uy = ua.y, uz = ua.z;
            const double g0 = tg[1 + 3 * a], g1 = tg[2 + 3 * a], g2 = tg[3 + 3 * a];
            x = x + g0 * ux;
            y = y + g1 * uy;
            z = z + g2 * uz;
            xy = xy + (g1 * ux + g0 * uy);
            yz = yz + (g2 * uy + g1 * uz);
            xz = xz + (g2 * ux + g0 * uz);
        }
        const double Vt = tg[0];
        tt[0] = Vt * x;
        tt[1] = Vt * y;
        tt[2] = Vt * z;
        tt[3] = Vt * xy;
        tt[4] = Vt * yz;
        tt[5] = Vt * xz;
    }
}

// the active elements of edge k in element order (hex e, then its remainder tets i): sum V, sum tau
// and (energy) the smoothing-domain volume sum V/n_e (R29)
__device__ __forceinline__ double edge_gather(const Dev &d, int64_t k, double *T, double *W) {
    const int64_t E = d.E;
    double Vh = 0.0, w = 0.0;
    // the edge's first four incidences in one 16-B load (a hex edge of a structured mesh has at most
    // four), gathered kHB at a time: state, V and the tau record of a pass in flight together; the
    // sums take them one after another in the incidence order.  Longer lists continue from the CSR.
    constexpr int kHB = CEM_HEXB_BATCH;  // 1, 2 or 4
    auto take = [&](const int32_t (&ent4)[kHB]) {
        uint8_t st4[kHB];
        double V4[kHB];
        double4 ta4[kHB];
        double2 tb4[kHB];
#pragma unroll
        for (int t = 0; t < kHB; ++t) {
            const int64_t e = ent4[t] >= 0 ? (int64_t)(ent4[t] >> 5) : 0;
            st4[t] = ent4[t] >= 0 ? __ldcg(d.state + e) : (uint8_t)0;
            V4[t] = __ldg(d.hgeo + e);
            ta4[t] = ldcg256h(reinterpret_cast<const double4 *>(d.htau) + e);
            tb4[t] = ldcg128h(reinterpret_cast<const double2 *>(d.htau + 4 * E) + e);
        }
#pragma unroll
        for (int t = 0; t < kHB; ++t) {
            if (ent4[t] < 0) break;
            const int64_t e = ent4[t] >> 5;
            const int pj = ent4[t] & 31;
            if (st4[t]) {
                if (c_hedge_of_pair[pj] < 0) continue;
                const double V = V4[t];
                Vh = Vh + V;
                if (W) w = w + V / 12.0;
                T[0] = T[0] + ta4[t].x;
                T[1] = T[1] + ta4[t].y;
                T[2] = T[2] + ta4[t].z;
                T[3] = T[3] + ta4[t].w;
                T[4] = T[4] + tb4[t].x;
                T[5] = T[5] + tb4[t].y;
                continue;
            }
            if (__ldcg(d.hrem + e) < 0) continue;
            const uint8_t ta = __ldcg(d.htact + e);
            for (int i = 0; i < 3; ++i) {
                if (!(ta >> i & 1) || !tet_has_pair(d.htloc + 12 * e + 4 * i, pj)) continue;
                const double V = __ldcg(d.htgeo + 39 * e + 13 * i);
                Vh = Vh + V;
                if (W) w = w + V / 6.0;
#pragma unroll
                for (int c = 0; c < 6; ++c) T[c] = T[c] + __ldcg(d.httau + 18 * e + 6 * i + c);
            }
        }
    };
    const int4 q4 = __ldg(d.heinc4 + k);
    const int32_t qq[4] = {q4.x, q4.y, q4.z, q4.w};
#pragma unroll
    for (int p = 0; p < 4 / kHB; ++p) {
        int32_t en[kHB];
#pragma unroll
        for (int t = 0; t < kHB; ++t) en[t] = qq[p * kHB + t];
        if (en[0] >= 0) take(en);
    }
    if (q4.w >= 0) {  // more than four incidences: the rest from the CSR
        const int32_t j1 = __ldg(d.e_off + k + 1);
        for (int32_t jn = __ldg(d.e_off + k) + 4; jn < j1; jn += kHB) {
            int32_t en[kHB];
#pragma unroll
            for (int t = 0; t < kHB; ++t) en[t] = jn + t < j1 ? __ldg(d.e_inc + jn + t) : -1;
            take(en);
        }
    }
    if (W) *W = w;
    return Vh;
}

// sigma record of edge k
__device__ __forceinline__ void hexB_edge(const Dev &d, int64_t k) {
    double T[6] = {0.0, 0.0, 0.0, 0.0, 0.0, 0.0};
    const double Vh = edge_gather(d, k, T, nullptr);
    double4 *o4 = reinterpret_cast<double4 *>(d.srec) + k;
    double2 *o2 = reinterpret_cast<double2 *>(d.srec2) + k;
    if (Vh == 0.0) {
        *o4 = make_double4(0.0, 0.0, 0.0, 0.0);
        *o2 = make_double2(0.0, 0.0);
        return;
    }
    const double inv = 1.0 / Vh;
    const double e11 = T[0] * inv, e22 = T[1] * inv, e33 = T[2] * inv, g12 = T[3] * inv, g23 = T[4] * inv,
                 g13 = T[5] * inv;
    *o4 = make_double4(d.l2m * e11 + d.lam * (e22 + e33), d.l2m * e22 + d.lam * (e11 + e33),
                       d.l2m * e33 + d.lam * (e11 + e22), d.mu * g12);
    *o2 = make_double2(d.mu * g23, d.mu * g13);
}

// blocks [0, ceil(S_h / 256)): one hex edge per thread.  Further blocks (launched once a crack step
// has run): the diagonal edges of the remainder prisms, from the list k_hexcrit appends to (a
// diagonal edge is carried by remainder tets only; the sigma record of an unlisted one stays the
// zero it was initialised to)
__global__ void __launch_bounds__(256, CEM_HEXB_BATCH >= 4 ? 2 : 4) k_hexB(Dev d, int64_t s) {
    pdl_trigger_h();
    const int nbh = (int)((d.hS_h + 255) / 256);
    if ((int)blockIdx.x < nbh) {
        const int64_t k = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
        if (k >= d.hS_h) return;
        pdl_wait_h();  // tau from stage A
        hexB_edge(d, k);
        return;
    }
    pdl_wait_h();
    const int n = __ldcg(d.ctr + 25);
    for (int i = ((int)blockIdx.x - nbh) * (int)blockDim.x + (int)threadIdx.x; i < n; i += ((int)gridDim.x - nbh) * (int)blockDim.x)
        hexB_edge(d, __ldcg(d.hdlist + i));
}

__device__ __forceinline__ void sigma_sum(const Dev &d, int32_t sid, double *S) {
    const double2 a0 = __ldcg(reinterpret_cast<const double2 *>(d.srec) + 2 * (int64_t)sid);
    const double2 a1 = __ldcg(reinterpret_cast<const double2 *>(d.srec) + 2 * (int64_t)sid + 1);
    const double2 b = __ldcg(reinterpret_cast<const double2 *>(d.srec2) + sid);
    S[0] = S[0] + a0.x;
    S[1] = S[1] + a0.y;
    S[2] = S[2] + a1.x;
    S[3] = S[3] + a1.y;
    S[4] = S[4] + b.x;
    S[5] = S[5] + b.y;
}

__global__ void __launch_bounds__(256) k_hexC(Dev d, int64_t s) {
    pdl_trigger_h();
    const int64_t E = d.E;
    const int64_t e = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (e >= E) return;
    int32_t sid[12];
#pragma unroll
    for (int l = 0; l < 12; ++l) sid[l] = __ldg(d.heedge + l * E + e);
    const double V = __ldg(d.hgeo + e);
    pdl_wait_h();  // sigma from stage B
    double4 *fo = reinterpret_cast<double4 *>(d.fe + 24 * e);  // slots 8e + a: 24 doubles, six 32-B stores
    double *fr = d.fe + 3 * (8 * E + 24 * e);                  // remainder slots 8E + 3(8e + a) + i at fr + 9a + 3i
    if (!__ldcg(d.state + e)) {
#pragma unroll
        for (int q = 0; q < 6; ++q) st256h(fo + q, 0.0, 0.0, 0.0, 0.0);
    } else {
        double S[6] = {0.0, 0.0, 0.0, 0.0, 0.0, 0.0};
#pragma unroll
        for (int l = 0; l < 12; ++l) sigma_sum(d, sid[l], S);
        const double c = V / 12.0;  // R26: the smoothing-domain share of each of the 12 edges
        double f[24];
#pragma unroll
        for (int a = 0; a < 8; ++a) {
            const double gx = __ldg(d.hgeo + (1 + 3 * a) * E + e), gy = __ldg(d.hgeo + (2 + 3 * a) * E + e),
                         gz = __ldg(d.hgeo + (3 + 3 * a) * E + e);
            f[3 * a] = c * ((gx * S[0] + gy * S[3]) + gz * S[5]);
            f[3 * a + 1] = c * ((gy * S[1] + gx * S[3]) + gz * S[4]);
            f[3 * a + 2] = c * ((gz * S[2] + gy * S[4]) + gx * S[5]);
        }
#pragma unroll
        for (int q = 0; q < 6; ++q) st256h(fo + q, f[4 * q], f[4 * q + 1], f[4 * q + 2], f[4 * q + 3]);
    }
    if (__ldcg(d.hrem + e) < 0) return;
    const uint8_t ta = __ldcg(d.htact + e);
    for (int i = 0; i < 3; ++i) {
        const uint8_t *tl = d.htloc + 12 * e + 4 * i;
        if (!(ta >> i & 1)) {  // a split tet contributes nothing from now on
            for (int b = 0; b < 4; ++b) {
                double *f = fr + 9 * tl[b] + 3 * i;
                f[0] = f[1] = f[2] = 0.0;
            }
            continue;
        }
        double S[6] = {0.0, 0.0, 0.0, 0.0, 0.0, 0.0};
        for (int l = 0; l < 6; ++l) sigma_sum(d, __ldg(d.hpair + (int64_t)c_hpair[tl[c_tp[l]]][tl[c_tq[l]]] * E + e), S);
        const double *tg = d.htgeo + 39 * e + 13 * i;
        const double c = tg[0] / 6.0;  // R5: V_t / 6 per tet edge
        for (int b = 0; b < 4; ++b) {
            const double gx = tg[1 + 3 * b], gy = tg[2 + 3 * b], gz = tg[3 + 3 * b];
            double *f = fr + 9 * tl[b] + 3 * i;
            f[0] = c * ((gx * S[0] + gy * S[3]) + gz * S[5]);
            f[1] = c * ((gy * S[1] + gx * S[3]) + gz * S[4]);
            f[2] = c * ((gz * S[2] + gy * S[4]) + gx * S[5]);
        }
    }
}

// strain energy of the edges of one 256-edge block on u_n (tau from k_hexA(n - 1)): psi(eps~_s)
// Vhat_s / 12 with psi = 1/2 lam tr^2 + mu eps:eps (the hex oracle's hx_strain_energy), summed by a
// fixed shuffle tree and the warps in order
__global__ void __launch_bounds__(256) k_hex_energy_edges(Dev d, double *part) {
    __shared__ double red[8];
    const int64_t S = d.S;
    const int64_t k = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    double U = 0.0;
    if (k < S) {
        double T[6] = {0, 0, 0, 0, 0, 0}, W = 0.0;
        const double Vh = edge_gather(d, k, T, &W);
        if (Vh != 0.0) {
            const double inv = 1.0 / Vh;
            const double e11 = T[0] * inv, e22 = T[1] * inv, e33 = T[2] * inv, g12 = T[3] * inv, g23 = T[4] * inv,
                         g13 = T[5] * inv;
            const double tr = e11 + e22 + e33;
            const double ee = e11 * e11 + e22 * e22 + e33 * e33 + 0.5 * (g12 * g12 + g23 * g23 + g13 * g13);
            U = (0.5 * d.lam * tr * tr + d.mu * ee) * W;
        }
    }
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) U = U + __shfl_down_sync(0xffffffffu, U, o);
    if ((threadIdx.x & 31) == 0) red[threadIdx.x >> 5] = U;
    __syncthreads();
    if (threadIdx.x == 0) {
        double t = 0.0;
        for (int i = 0; i < (int)(blockDim.x >> 5); ++i) t = t + red[i];
        part[blockIdx.x] = t;
    }
}

template <class K, class... Args>
void launch_pdl_h(K kern, unsigned grid, cudaStream_t st, Args... args) {
    cudaLaunchConfig_t cfg = {};
    cfg.gridDim = dim3(grid);
    cfg.blockDim = dim3(256);
    cfg.stream = st;
    cudaLaunchAttribute at[1];
    at[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
    at[0].val.programmaticStreamSerializationAllowed = 1;
    cfg.attrs = at;
    cfg.numAttrs = 1;
    cudaLaunchKernelEx(&cfg, kern, args...);
}

}  // namespace

void launch_hex_energy(const Dev &d, int64_t n, double *part_edges, double *part_nodes, cudaStream_t st) {
    const unsigned ge = (unsigned)((d.E + 255) / 256), gs = (unsigned)((d.S + 255) / 256);
    k_hexA<<<ge, 256, 0, st>>>(d, n - 1);  // tau of u_n = ubuf[n & 1]
    k_hex_energy_edges<<<gs, 256, 0, st>>>(d, part_edges);
    launch_energy_nodes(d, n, part_nodes, st);
}

int launch_hex_step(const Dev &d, int64_t s, cudaStream_t st, bool crack, bool diagonals) {
    // stage B's grid has blocks for the listed diagonal edges (carried by remainder tets only) once a
    // crack step has run in this context (`diagonals`, host-known); before that no remainder can exist
    const unsigned ge = (unsigned)((d.E + 255) / 256), gs = (unsigned)((d.hS_h + 255) / 256) + (diagonals ? 148u * 4u : 0u);
    launch_pdl_h(k_hexA, ge, st, d, s);
    launch_pdl_h(k_hexB, gs, st, d, s);
    launch_pdl_h(k_hexC, ge, st, d, s);
    if (crack) launch_hex_crit(d, s, st);
    launch_node_update(d, s, st);
    return crack ? 6 : 4;
}

}  // namespace cem
